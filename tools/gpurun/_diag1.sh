mkdir -p gpurun_out/d1
timeout 600 python tools/pipe_ab.py --experts 128 --reps 5 --steps 8 > gpurun_out/d1/pipe_ab.txt 2>&1
timeout 300 python tools/timeline.py --experts 128 --budget-frac 1.0 --steps 4 --warmup 6 --out gpurun_out/d1/tl100.json > gpurun_out/d1/tl100.txt 2>&1
timeout 300 python tools/timeline.py --experts 128 --budget-frac 0.97 --steps 4 --warmup 6 --out gpurun_out/d1/tl097.json > gpurun_out/d1/tl097.txt 2>&1
cat gpurun_out/d1/*.txt
