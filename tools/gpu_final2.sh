timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "fused" 2>&1 | tail -2
timeout 900 python bench.py > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
tail -2 gpurun_out/bench_c2.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/b_ncu.log 2>&1
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:k_nbrscore --launch-skip 1 -c 1 -o gpurun_out/nbr_full python tools/run_level.py --steps 1 > gpurun_out/ncu_nbr.log 2>&1
python tools/ncu_summary.py gpurun_out/nbr_full.ncu-rep > gpurun_out/nbr_summary.txt 2>&1
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -1 gpurun_out/smoke.log
cat gpurun_out/bench_c2.json
