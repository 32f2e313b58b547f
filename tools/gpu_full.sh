# full round evidence: GPU tests, default bench line, launch list (ncu, timing pass), ncu --set full of the top kernel
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
timeout 1800 python -m pytest tests -m gpu -x -q 2>&1 | tail -5 > gpurun_out/pytest_gpu.log
cat gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
tail -2 gpurun_out/bench_c2.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/b_ncu.log 2>&1
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:k_nbrscore -c 1 -o gpurun_out/nbr_full python tools/run_level.py --steps 1 > gpurun_out/ncu_nbr.log 2>&1
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -2 gpurun_out/smoke.log
python tools/ncu_summary.py gpurun_out/nbr_full.ncu-rep > gpurun_out/nbr_summary.txt 2>&1
cat gpurun_out/bench_c2.json
bash tools/gpu_workloads.sh > gpurun_out/workloads.txt 2>&1
cat gpurun_out/workloads.txt
