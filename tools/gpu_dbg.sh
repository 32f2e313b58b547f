HGP_DEBUG_SYNC=1 timeout 300 python tools/run_level.py --steps 1 > gpurun_out/dbg.log 2>&1
echo rc=$?
tail -30 gpurun_out/dbg.log
