# Round-end evidence on one B200: GPU tests, smoke, bench line, launch list of a short bench,
# ncu --set full of one layer's FFN GEMMs (base-8 and base-128) and the attention kernels.
set -x
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gputests.log 2>&1; echo tests=$?
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
timeout 600 python bench.py > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bench.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-streaming --no-north-star > /dev/null 2>&1
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:"grouped_gemm" -s 4 -c 2 --csv python tools/ffn_probe.py --iters 2 --no-cublas > gpurun_out/ffn8_traffic.csv 2>&1
ncu --set full --import-source on --clock-control none -k regex:"grouped_gemm" -s 4 -c 2 -o gpurun_out/ffn8_full python tools/ffn_probe.py --iters 2 --no-cublas > /dev/null 2>&1
ncu --set full --import-source on --clock-control none -k regex:"grouped_gemm" -s 4 -c 2 -o gpurun_out/ffn128_full python tools/ffn_probe.py --experts 128 --iters 2 --no-cublas > /dev/null 2>&1
ncu --set full --import-source on --clock-control none -k regex:"grouped_gemm|attn_core" -s 6 -c 4 -o gpurun_out/layer_full python tools/attn_probe.py --iters 2 > /dev/null 2>&1
tail -3 gpurun_out/gputests.log; tail -2 gpurun_out/smoke.log
ls -la gpurun_out
