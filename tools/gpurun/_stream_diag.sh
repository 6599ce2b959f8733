mkdir -p gpurun_out/sd
for bf in 1.0 0.97; do for pol in spread fifo; do timeout 300 python tools/host_time.py --experts 128 --budget-frac $bf --victim-policy $pol; done; done > gpurun_out/sd/host.txt 2>&1
timeout 300 python tools/timeline.py --experts 128 --budget-frac 0.97 --steps 4 --warmup 6 --out gpurun_out/sd/tl097.json > gpurun_out/sd/tl097.txt 2>&1
timeout 300 python tools/timeline.py --experts 128 --budget-frac 1.0 --steps 4 --warmup 6 --out gpurun_out/sd/tl100.json > gpurun_out/sd/tl100.txt 2>&1
cat gpurun_out/sd/*.txt
