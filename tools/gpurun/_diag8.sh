mkdir -p gpurun_out/d8
{
python tools/permute_probe.py
python tools/permute_probe.py --rows 32768 --experts 128
python tools/permute_probe.py --rows 32768 --experts 8
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider 2>&1 | tail -3
N="ncu --set full --import-source on --clock-control none"
timeout 600 $N -k regex:"rank_tiles|tile_base|place_tiles" -s 3 -c 3 -o gpurun_out/d8/permute_c4_full python tools/permute_probe.py > /dev/null 2>&1
timeout 600 $N -k regex:"rank_tiles|tile_base|place_tiles" -s 3 -c 3 -o gpurun_out/d8/permute_bench_full python tools/permute_probe.py --rows 32768 --experts 128 > /dev/null 2>&1
} > gpurun_out/d8/out.txt 2>&1
cat gpurun_out/d8/out.txt
