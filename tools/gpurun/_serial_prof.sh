# host profile of serve_sida with the hash on the compute stream (SIDA_HASH_SERIAL=1)
mkdir -p gpurun_out/ser
SIDA_HASH_SERIAL=1 timeout 300 python tools/e2e_probe.py --batches 20 --reps 1 2>&1 | tee gpurun_out/ser/prof_serial.txt
