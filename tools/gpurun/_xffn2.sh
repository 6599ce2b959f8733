mkdir -p gpurun_out/x2
for m in 5 1 0; do echo "mode $m"; timeout 120 python tools/xffn_debug.py $m; done > gpurun_out/x2/debug.txt 2>&1
for e in 8 128; do timeout 120 python tools/ffn_probe.py --experts $e --no-cublas; done > gpurun_out/x2/probe.txt 2>&1
for lag in 13 40 80; do SIDA_XFFN_LAG=$lag timeout 120 python tools/ffn_probe.py --experts 128 --no-cublas; done >> gpurun_out/x2/probe.txt 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"expert_ffn" -s 2 -c 1 -o gpurun_out/x2/xffn128 python tools/ffn_probe.py --experts 128 --iters 2 --no-cublas > /dev/null 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"expert_ffn" -s 2 -c 1 -o gpurun_out/x2/xffn8 python tools/ffn_probe.py --experts 8 --iters 2 --no-cublas > /dev/null 2>&1
cat gpurun_out/x2/debug.txt gpurun_out/x2/probe.txt
