for r in 1 2; do for v in 0 1; do echo "== rev $v"; SIDA_FFN_REV2=$v python tools/ffn_probe.py --experts 128 --iters 30 --no-cublas; SIDA_FFN_REV2=$v python tools/ffn_probe.py --experts 8 --iters 30 --no-cublas; done; done
timeout 600 python -m pytest tests/test_gpu_kernels.py -q -x -p no:cacheprovider -k "ffn" 2>&1 | tail -1
