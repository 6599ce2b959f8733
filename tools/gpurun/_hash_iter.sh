# hash kernels: bit-exactness tests + timings + launch list
mkdir -p gpurun_out/h
timeout 900 python -m pytest tests/test_gpu_kernels.py -q -x -k "hash" -p no:cacheprovider > gpurun_out/h/tests.log 2>&1; echo tests=$?
for e in 8 64 128; do python tools/hash_probe.py --experts $e; SIDA_HASH_HEADS_SPLIT=0 python tools/hash_probe.py --experts $e; done > gpurun_out/h/probe.txt 2>&1
python tools/hash_probe.py --experts 128 --seq 512 --batch 64 >> gpurun_out/h/probe.txt 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/h/launches.csv python tools/hash_probe.py --experts 128 --iters 3 > /dev/null 2>&1
python tools/launch_share.py gpurun_out/h/launches.csv > gpurun_out/h/share.txt
tail -3 gpurun_out/h/tests.log; cat gpurun_out/h/probe.txt gpurun_out/h/share.txt
