# Per-CTA GEMM counters: static-schedule imbalance of the FFN GEMMs (base-128, 32K rows)
mkdir -p gpurun_out/sp
SIDA_GEMM_PROF=1 timeout 120 python tools/ffn_probe.py --experts 128 --no-cublas > gpurun_out/sp/prof.txt 2>&1
SIDA_GEMM_PROF=1 timeout 120 python tools/ffn_probe.py --experts 128 --no-cublas --exact >> gpurun_out/sp/prof.txt 2>&1
cat gpurun_out/sp/prof.txt
