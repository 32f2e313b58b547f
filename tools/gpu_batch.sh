cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout 2400 python -m pytest tests/test_gpu_shard.py tests/test_gpu_tiers.py tests/test_gpu_multilevel.py tests/test_gpu_golden.py "tests/test_gpu_parity.py::test_level_steps_match_oracle" -x -q --durations=8 > gpurun_out/pytest_quick.log 2>&1; grep -E "never exercised|passed|failed|Error|s call" gpurun_out/pytest_quick.log | head -30
