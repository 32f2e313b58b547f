cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -k "fused or giant or level_steps" -x -q > gpurun_out/pytest_quick.log 2>&1; tail -3 gpurun_out/pytest_quick.log
BENCH_ARGS="--no-refine --no-e2e --steps 3" bash tools/gpu.sh bench
timeout 1500 python bench.py --workload C5 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-hier > gpurun_out/bench_C5.json 2> gpurun_out/bench_C5.err; echo "bench rc=$?"; tail -3 gpurun_out/bench_C5.err
python tools/bench_brief.py gpurun_out/bench_C5.json
