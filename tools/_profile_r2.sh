# Round-2 evidence on one B200: the launch list of a short bench and ncu --set full of the
# hot kernels at the bench shape (tests/smoke/bench run separately: tools/_gpu_quick.sh).
mkdir -p gpurun_out/r2
N="ncu --set full --import-source on --clock-control none"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2/launches_bench.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-extras > gpurun_out/r2/launches_bench.log 2>&1; echo launches=$?
timeout 900 $N -k regex:"grouped_gemm" -s 4 -c 2 -o gpurun_out/r2/ffn128_full python tools/ffn_probe.py --experts 128 --iters 3 --no-cublas > /dev/null 2>&1; echo ffn128=$?
timeout 900 $N -k regex:"grouped_gemm|attn_core|qkv" -s 6 -c 4 -o gpurun_out/r2/attn128_full python tools/attn_probe.py --iters 3 > /dev/null 2>&1; echo attn=$?
timeout 900 $N -k regex:"rank_tiles|tile_base|place_tiles" -s 2 -c 2 -o gpurun_out/r2/permute_c4_full python tools/permute_probe.py > /dev/null 2>&1; echo perm=$?
timeout 900 $N -k regex:"rank_tiles|tile_base|place_tiles" -s 2 -c 2 -o gpurun_out/r2/permute_bench_full python tools/permute_probe.py --rows 32768 --experts 128 > /dev/null 2>&1; echo perm2=$?
timeout 900 $N -k regex:"lstm|rows_dmma|attn_block|project" -s 0 -c 6 -o gpurun_out/r2/hash128_full python tools/hash_probe.py --experts 128 > gpurun_out/r2/hash_probe.log 2>&1; echo hash=$?
ls -la gpurun_out/r2
