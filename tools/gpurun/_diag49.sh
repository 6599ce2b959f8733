for S in 1 2 4; do echo "S=$S $(SIDA_LSTM_S=$S python tools/hash_probe.py --experts 128 2>&1 | tail -1)"; SIDA_LSTM_S=$S python tools/pipe_ab.py --modes flat --reps 3 --steps 10 2>&1 | tail -1; done
SIDA_LSTM_S=2 timeout 300 python -m pytest tests/test_gpu_kernels.py -q -x -p no:cacheprovider -k "hash" 2>&1 | tail -1
