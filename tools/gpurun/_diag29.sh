mkdir -p gpurun_out/d29
SIDA_FFN_TS=1 timeout 600 ncu --set full --import-source on --clock-control none -k regex:"ffn1_ts" -s 2 -c 1 -o gpurun_out/d29/ts8 python tools/ffn_probe.py --experts 8 --iters 3 --no-cublas > /dev/null 2>&1; echo ncu=$?
