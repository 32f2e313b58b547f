# quick GPU iteration: fused-path parity + bench (no e2e / cpu baseline)
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_multilevel.py -m gpu -x -q -k "fused or giant or level_steps or multilevel" 2>&1 | tail -4 > gpurun_out/pytest_quick.log
cat gpurun_out/pytest_quick.log
timeout 600 python bench.py --no-cpu-baseline --no-e2e ${BENCH_ARGS} > gpurun_out/bench_quick.json 2> gpurun_out/bench_quick.err
tail -2 gpurun_out/bench_quick.err
python -c "
import json; d=json.load(open('gpurun_out/bench_quick.json'))
print('ms/step', round(d['ms_per_step'],3), 'pins/s %.3e'%d['value']); print(d['step_ms']); print(d['kernels_ms'])"
