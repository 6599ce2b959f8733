SIDA_OUTPROJ_TN=1 timeout 600 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "proj or c1" 2>&1 | tail -2
for r in 1 2; do for v in 0 1; do echo "tn=$v $(SIDA_OUTPROJ_TN=$v python tools/attn_probe.py 2>&1 | tail -1)"; done; done
for v in 0 1; do echo "tn=$v $(SIDA_OUTPROJ_TN=$v python tools/fwd_probe.py --steps 8 2>&1 | tail -2 | head -1)"; done
