for r in 1 2; do for bn in 192 256 128; do echo "bn=$bn $(SIDA_OUTPROJ_BN=$bn python tools/attn_probe.py 2>&1 | tail -1)"; done; done
