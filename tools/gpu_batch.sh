cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -k "fused or giant" -x -q 2>&1 | tail -5 > gpurun_out/pytest_quick.log; cat gpurun_out/pytest_quick.log
BENCH_ARGS="--no-refine --no-e2e --steps 3" bash tools/gpu.sh bench
NCU_K=k_nbrscore NCU_SKIP=1 NCU_OUT=nbrscore6 bash tools/gpu.sh ncu
