mkdir -p gpurun_out/x3
for m in 5 0; do echo "mode $m"; timeout 120 python tools/xffn_debug.py $m; done > gpurun_out/x3/debug.txt 2>&1
timeout 300 python -m pytest tests/test_gpu_kernels.py -q -x -k "one_launch" -p no:cacheprovider 2>&1 | tail -3 >> gpurun_out/x3/debug.txt
for e in 8 128; do for lag in 25 80; do SIDA_XFFN_LAG=$lag SIDA_XFFN_PROF=1 timeout 120 python tools/ffn_probe.py --experts $e --no-cublas --iters 3; done; done > gpurun_out/x3/probe.txt 2>&1
cat gpurun_out/x3/debug.txt gpurun_out/x3/probe.txt
