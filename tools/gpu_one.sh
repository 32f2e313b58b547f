timeout 1500 python -m pytest tests/test_gpu_fullsize.py tests/test_gpu_shard.py -m gpu -q 2>&1 | tail -2
