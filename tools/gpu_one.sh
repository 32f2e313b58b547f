timeout 1800 python -m pytest tests/test_gpu_parity.py tests/test_gpu_multilevel.py tests/test_gpu_leftover.py -m gpu -x -q 2>&1 | tail -2
timeout 900 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_q.json 2> gpurun_out/bench_q.err
python -c "
import json; d=json.load(open('gpurun_out/bench_q.json'))
print('ms/step', round(d['ms_per_step'],3), 'pins/s %.3e'%d['value']); print(d['step_ms']); h=d['hierarchy']; print('hier', h['total_coarsening_ms'], h['levels'], h['level_ms'][:6])"
