timeout 600 python -m pytest tests/test_gpu_pipeline_contracts.py tests/test_gpu_parity.py -q -x -p no:cacheprovider 2>&1 | tail -2
