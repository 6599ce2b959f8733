for E in 128 8; do SIDA_GEMM_PROF=1 python tools/ffn_probe.py --experts $E --iters 20 --no-cublas 2>&1 | head -8; done
SIDA_GEMM_PROF=1 python tools/ffn_probe.py --experts 128 --iters 20 --no-cublas --exact 2>&1 | head -8
