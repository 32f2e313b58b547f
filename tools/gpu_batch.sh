cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_tiers.py -k "fused or level_steps" -x -q > gpurun_out/pytest_quick.log 2>&1; tail -3 gpurun_out/pytest_quick.log
for wl in C4 C3; do
  timeout 1200 python bench.py --workload $wl --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-hier > gpurun_out/bench_$wl.json 2> gpurun_out/bench_$wl.err
  echo "== $wl rc=$?"; tail -2 gpurun_out/bench_$wl.err; python tools/bench_brief.py gpurun_out/bench_$wl.json
done
