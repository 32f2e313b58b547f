# bench lines for the other BASELINE configs (quick: no cpu baseline / e2e)
for wl in C2r C3 C4; do
  timeout 900 python bench.py --workload $wl --no-cpu-baseline --no-e2e > gpurun_out/bench_$wl.json 2> gpurun_out/bench_$wl.err
  echo "== $wl rc=$?"; tail -1 gpurun_out/bench_$wl.err
  python -c "
import json; d=json.load(open('gpurun_out/bench_$wl.json'))
print('ms/step', round(d['ms_per_step'],3), 'pins/s %.3e'%d['value'], 'V', d['config']['V']); print(d['step_ms']); print(list(d['kernels_ms'].items())[:6]); h=d.get('hierarchy'); print('hier', h and (round(h['total_coarsening_ms'],1), h['levels']))"
done
