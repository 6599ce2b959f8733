timeout 600 python -m pytest tests/test_gpu_kernels.py -q -x -p no:cacheprovider -k "ffn or linear or out_proj" 2>&1 | tail -2
AB_CMD='for E in 128 8; do python tools/ffn_probe.py --experts $E --iters 30 --no-cublas; done; python tools/attn_probe.py 2>&1 | tail -1' bash tools/_ab.sh
