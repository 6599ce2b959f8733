export SIDA_FFN_TS=1
timeout 300 python tools/ffn_probe.py --experts 8 --iters 5 --no-cublas; echo probe=$?
timeout 600 python -m pytest tests/test_gpu_kernels.py -q -x -p no:cacheprovider -k "grouped_ffn_bf16_vs_oracle and (-1-)" 2>&1 | tail -3
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "north_star" 2>&1 | tail -3
for E in 128 8 64; do echo "== TS $E"; timeout 300 python tools/ffn_probe.py --experts $E --iters 20 --no-cublas; echo "== base $E"; SIDA_FFN_TS=0 timeout 300 python tools/ffn_probe.py --experts $E --iters 20 --no-cublas; done
