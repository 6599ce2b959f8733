mkdir -p gpurun_out/d6
{
timeout 300 python tools/fwd_probe.py --experts 128
timeout 300 python tools/host_time.py --experts 128 --budget-frac 1.0
timeout 300 python tools/host_time.py --experts 128 --budget-frac 0.97
} > gpurun_out/d6/out.txt 2>&1
cat gpurun_out/d6/out.txt
