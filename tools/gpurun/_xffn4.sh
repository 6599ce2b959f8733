mkdir -p gpurun_out/x4
timeout 300 python -m pytest tests/test_gpu_kernels.py -q -x -k "one_launch or (ffn_bf16_vs_oracle and 5)" -p no:cacheprovider 2>&1 | tail -2 > gpurun_out/x4/tests.txt
for e in 8 128; do for lag in 25 80; do SIDA_XFFN_LAG=$lag SIDA_XFFN_PROF=1 timeout 120 python tools/ffn_probe.py --experts $e --no-cublas --iters 10; done; SIDA_XFFN=0 timeout 120 python tools/ffn_probe.py --experts $e --no-cublas --iters 10; done > gpurun_out/x4/probe.txt 2>&1
cat gpurun_out/x4/tests.txt gpurun_out/x4/probe.txt
