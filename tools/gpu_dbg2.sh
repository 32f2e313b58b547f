timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_multilevel.py -m gpu -x -q 2>&1 | tail -4 > gpurun_out/pytest_dbg2.log
cat gpurun_out/pytest_dbg2.log
HGP_DEBUG_SYNC=1 timeout 300 python tools/run_level.py --steps 2 > gpurun_out/dbg2.log 2>&1
grep -E "radix|inc_|score_|nbrscore|coarse_nbrs|segsort" gpurun_out/dbg2.log | tail -40
