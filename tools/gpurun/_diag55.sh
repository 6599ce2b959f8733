timeout 600 python -m pytest tests/test_gpu_serving.py tests/test_gpu_pipeline_contracts.py -q -x -p no:cacheprovider 2>&1 | tail -1
bash tools/gpurun/_diag36.sh
