mkdir -p gpurun_out/d4
N="ncu --set full --import-source on --clock-control none"
SIDA_XFFN=1 timeout 600 $N -k regex:"expert_ffn|gather|memset|fill" -s 3 -c 3 -o gpurun_out/d4/xffn128 python tools/ffn_probe.py --experts 128 --iters 3 --no-cublas > gpurun_out/d4/xffn.log 2>&1
SIDA_FFN_SWAP=1 timeout 600 $N -k regex:"gemm" -s 4 -c 2 -o gpurun_out/d4/tn128 python tools/ffn_probe.py --experts 128 --iters 3 --no-cublas > gpurun_out/d4/tn.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/d4/xffn_launches.csv env SIDA_XFFN=1 python tools/ffn_probe.py --experts 128 --iters 3 --no-cublas > /dev/null 2>&1
echo done
