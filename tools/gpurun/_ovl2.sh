mkdir -p gpurun_out/ov2
timeout 300 python -m pytest tests/test_gpu_kernels.py -q -x -k "hash" -p no:cacheprovider 2>&1 | tail -1
for cfg in "SIDA_HEADS_SPLIT_Y=1" "SIDA_HEADS_SPLIT_Y=0" "SIDA_LSTM_CHUNK=16" "SIDA_LSTM_CHUNK=32" "SIDA_LSTM_CHUNK=8"; do echo "$cfg"; env $cfg timeout 300 python tools/overlap_probe.py --experts 128; done 2>&1
