timeout 1800 python -m pytest tests/test_gpu_parity.py tests/test_gpu_multilevel.py -m gpu -x -q 2>&1 | tail -3
for wl in C2 C2r; do
timeout 900 python bench.py --workload $wl --no-cpu-baseline --no-e2e > gpurun_out/bench_q.json 2> gpurun_out/bench_q.err
tail -1 gpurun_out/bench_q.err
python -c "
import json; d=json.load(open('gpurun_out/bench_q.json'))
print('$wl ms/step', round(d['ms_per_step'],3), 'pins/s %.3e'%d['value']); print(d['step_ms']); print(list(d['kernels_ms'].items())[:8]); h=d['hierarchy']; print('hier', h['total_coarsening_ms'], h['levels'], h['level_ms'][:6])"
done
