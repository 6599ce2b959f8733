mkdir -p gpurun_out/ser
SIDA_HASH_SERIAL=1 timeout 300 python tools/serial_probe.py 2>&1 | tee gpurun_out/ser/timeline_serial.txt
timeout 300 python tools/serial_probe.py 2>&1 | tee gpurun_out/ser/timeline_overlap.txt
