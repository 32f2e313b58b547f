HGP_DEBUG_SYNC=1 timeout 300 python tools/run_level.py --steps 2 > gpurun_out/dbg3.log 2>&1
awk '/radix|inc_|segsort|score_|nbrscore|coarse_nbrs|cnbr|edge_unique|merge|map_pins/' gpurun_out/dbg3.log | tail -32
timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_q.json 2> gpurun_out/bench_q.err
python -c "
import json; d=json.load(open('gpurun_out/bench_q.json'))
print('ms/step', round(d['ms_per_step'],3), 'pins/s %.3e'%d['value']); print(d['step_ms']); print(d['kernels_ms']); h=d['hierarchy']; print('hier', h['total_coarsening_ms'], h['levels'], h['level_ms'][:6])"
