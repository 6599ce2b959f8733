# Hash overlapped on its own stream (default) vs hash on the compute stream (SIDA_HASH_SERIAL=1): per-batch device latency
mkdir -p gpurun_out/ser
for r in 1 2; do
for s in "" 1; do
  echo "== serial=$s run $r"
  SIDA_HASH_SERIAL=$s timeout 300 python tools/e2e_probe.py --batches 20 --reps 2 2>&1 | grep "^rep"
done
done 2>&1 | tee gpurun_out/ser/probe.txt
