mkdir -p gpurun_out/ov
python tools/overlap_probe.py --experts 128 > gpurun_out/ov/a.txt 2>&1
SIDA_HASH_SERIAL=1 python tools/overlap_probe.py --experts 128 > gpurun_out/ov/serial.txt 2>&1
SIDA_FLAT_PRIORITY=1 python tools/overlap_probe.py --experts 128 > gpurun_out/ov/flat.txt 2>&1
SIDA_HASH_PROF=1 python tools/hash_probe.py --experts 128 > gpurun_out/ov/hashprof.txt 2>&1
python tools/hash_probe.py --experts 8 > gpurun_out/ov/hash8.txt 2>&1
cat gpurun_out/ov/*.txt
