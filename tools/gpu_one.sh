timeout 300 python tools/bisect/diff_cand.py 2>&1 | tail -3
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_multilevel.py -m gpu -x -q 2>&1 | tail -3
