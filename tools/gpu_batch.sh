cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_multilevel.py -k "level_steps or composition or multilevel or hierarch" -x -q 2>&1 | tail -5 > gpurun_out/pytest_quick.log; cat gpurun_out/pytest_quick.log
BENCH_ARGS="--no-refine --no-e2e --steps 3" bash tools/gpu.sh bench
NCU_K=k_score_flat NCU_SKIP=0 NCU_OUT=scoreflat4 NCU_ARGS=--hierarchy bash tools/gpu.sh ncu
