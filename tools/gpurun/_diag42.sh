mkdir -p gpurun_out/d42
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"heads_dmma|attn_block|lstm_quad" -s 3 -c 4 -o gpurun_out/d42/hash python tools/hash_probe.py --experts 128 > /dev/null 2>&1; echo ncu=$?
