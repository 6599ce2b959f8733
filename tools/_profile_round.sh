set -x
timeout 600 python bench.py > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bench.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-streaming > /dev/null 2>&1
ncu --set full --import-source on --clock-control none -k regex:"grouped_gemm|attn_core" -s 6 -c 4 -o gpurun_out/layer_full python tools/attn_probe.py --iters 2 > /dev/null 2>&1
ncu --set full --import-source on --clock-control none -k regex:"grouped_gemm" -s 4 -c 2 -o gpurun_out/ffn8_full python tools/ffn_probe.py --iters 2 --no-cublas > /dev/null 2>&1
ls -la gpurun_out
