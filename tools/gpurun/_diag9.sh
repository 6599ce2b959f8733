mkdir -p gpurun_out/d9
{
python tools/permute_probe.py
python tools/permute_probe.py --rows 32768 --experts 128
timeout 900 python -m pytest tests/test_gpu_kernels.py -q -x -p no:cacheprovider -k "permute or hash" 2>&1 | tail -2
N="ncu --set full --import-source on --clock-control none"
timeout 600 $N -k regex:"rank_tiles|tile_base|place_tiles" -s 3 -c 3 -o gpurun_out/d9/permute_c4_full python tools/permute_probe.py > /dev/null 2>&1
timeout 600 $N -k regex:"rank_tiles|tile_base|place_tiles" -s 3 -c 3 -o gpurun_out/d9/permute_bench_full python tools/permute_probe.py --rows 32768 --experts 128 > /dev/null 2>&1
echo "== xffn normal"; SIDA_XFFN=1 SIDA_XFFN_PROF=1 python tools/ffn_probe.py --experts 128 --iters 20 --no-cublas
echo "== xffn diag1"; SIDA_XFFN=1 SIDA_XFFN_DIAG=1 SIDA_XFFN_PROF=1 python tools/ffn_probe.py --experts 128 --iters 20 --no-cublas
echo "== xffn diag1 alias"; SIDA_XFFN=1 SIDA_XFFN_DIAG=1 SIDA_XFFN_PROF=1 python tools/ffn_probe.py --experts 128 --iters 20 --no-cublas --alias-slots 4
echo "== xffn 8"; SIDA_XFFN=1 python tools/ffn_probe.py --experts 8 --iters 20 --no-cublas
} > gpurun_out/d9/out.txt 2>&1
cat gpurun_out/d9/out.txt
