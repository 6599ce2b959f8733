mkdir -p gpurun_out/hn
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"heads_dmma|attn_block|lstm_quad" -s 4 -c 4 -o gpurun_out/hn/hash128 python tools/hash_probe.py --experts 128 --iters 2 > gpurun_out/hn/log.txt 2>&1
tail -3 gpurun_out/hn/log.txt
