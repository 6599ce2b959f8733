# one-launch expert FFN: parity tests + timings vs the two-launch path
mkdir -p gpurun_out/x
timeout 300 python tools/ffn_probe.py --experts 128 --iters 5 --no-cublas > gpurun_out/x/smoke.txt 2>&1; echo smoke=$?
cat gpurun_out/x/smoke.txt
timeout 600 python -m pytest tests/test_gpu_kernels.py -q -x -k "ffn" -p no:cacheprovider > gpurun_out/x/tests.log 2>&1; echo tests=$?
tail -15 gpurun_out/x/tests.log
for e in 8 64 128 256; do timeout 120 python tools/ffn_probe.py --experts $e --no-cublas; SIDA_XFFN=0 timeout 120 python tools/ffn_probe.py --experts $e --no-cublas; done > gpurun_out/x/probe.txt 2>&1
timeout 120 python tools/ffn_probe.py --experts 128 --tokens 131072 --no-cublas >> gpurun_out/x/probe.txt 2>&1
SIDA_XFFN=0 timeout 120 python tools/ffn_probe.py --experts 128 --tokens 131072 --no-cublas >> gpurun_out/x/probe.txt 2>&1
cat gpurun_out/x/probe.txt
