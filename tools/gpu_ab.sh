# parity of a1/fused paths + A/B bench variants
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_multilevel.py tests/test_gpu_fullsize.py -m gpu -x -q 2>&1 | tail -4 > gpurun_out/pytest_ab.log
cat gpurun_out/pytest_ab.log
for v in "" "HGP_INC_ATOMIC=1" "HGP_FUSED_CFG=2"; do
  env $v timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_ab.json 2> gpurun_out/bench_ab.err
  echo "== $v"; tail -1 gpurun_out/bench_ab.err
  python -c "
import json; d=json.load(open('gpurun_out/bench_ab.json'))
print('ms/step', round(d['ms_per_step'],3), 'pins/s %.3e'%d['value'], 'hier', d.get('hierarchy',{}).get('total_coarsening_ms')); print(d['step_ms']); print(d['kernels_ms'])"
done
