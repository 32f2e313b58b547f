timeout 1800 python -m pytest tests/test_gpu_parity.py tests/test_gpu_multilevel.py tests/test_gpu_leftover.py -m gpu -x -q 2>&1 | tail -2
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
