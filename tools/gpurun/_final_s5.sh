# final-tree evidence: tests, smoke, bench (both arms), attention/out-projection ncu
bash tools/_gpu_quick.sh
mkdir -p gpurun_out/r2
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"grouped_gemm|attn_core" -s 6 -c 4 -o gpurun_out/r2/attn128_full_s5 python tools/attn_probe.py --iters 3 > /dev/null 2>&1; echo attn=$?
