# Round-2 evidence on one B200: GPU tests, smoke, the bench line, the launch list of a
# short bench, ncu --set full of the hot kernels at the bench shape, the overlap timeline.
set -x
mkdir -p gpurun_out/r2
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r2/gputests.log 2>&1; echo tests=$?
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2/smoke.log 2>&1; echo smoke=$?
timeout 900 python bench.py > gpurun_out/r2/bench.json 2> gpurun_out/r2/bench.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r2/bench_ref.json 2> gpurun_out/r2/bench_ref.err
timeout 300 python tools/timeline.py --out gpurun_out/r2/timeline_097.json > gpurun_out/r2/timeline_097.txt 2>&1
timeout 300 python tools/timeline.py --budget-frac 0.9 --out gpurun_out/r2/timeline_090.json > gpurun_out/r2/timeline_090.txt 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2/launches_bench.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-extras > /dev/null 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"grouped_gemm" -s 4 -c 2 -o gpurun_out/r2/ffn128_full python tools/ffn_probe.py --experts 128 --iters 2 --no-cublas > /dev/null 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"grouped_gemm" -s 4 -c 2 -o gpurun_out/r2/ffn8_full python tools/ffn_probe.py --experts 8 --iters 2 --no-cublas > /dev/null 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"grouped_gemm|attn_core" -s 6 -c 3 -o gpurun_out/r2/attn128_full python tools/attn_probe.py --iters 2 > /dev/null 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"attn_core" -s 2 -c 1 -o gpurun_out/r2/attn512_full python tools/attn_probe.py --batch 64 --seq 512 --iters 2 > /dev/null 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"hist_tiles|scatter_kernel|gather_rows" -s 3 -c 3 -o gpurun_out/r2/permute_c4_full python tools/permute_probe.py > /dev/null 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"hist_tiles|scatter_kernel" -s 2 -c 2 -o gpurun_out/r2/permute_bench_full python tools/permute_probe.py --rows 32768 --experts 128 > /dev/null 2>&1
tail -3 gpurun_out/r2/gputests.log; tail -2 gpurun_out/r2/smoke.log
ls -la gpurun_out/r2
