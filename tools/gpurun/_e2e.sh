# Where the e2e (serve_sida, host batches) wall clock goes at the bench shape: per-call overhead vs batches per call
mkdir -p gpurun_out/e2e
for nb in 10 30; do timeout 300 python tools/e2e_probe.py --batches $nb --reps 3; done 2>&1 | tee gpurun_out/e2e/probe.txt
