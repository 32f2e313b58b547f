#!/bin/bash
# One gpurun call = one or more of these steps, in order:  bash tools/gpu.sh tests bench ncu ...
#   tests      pytest -m gpu (all)                 -> gpurun_out/pytest_gpu.log
#   tq         pytest -m gpu -k "$PYK"             -> gpurun_out/pytest_quick.log
#   bench      bench.py (C2, no cpu baseline)      -> gpurun_out/bench_c2.json
#   benchfull  bench.py (C2, everything)           -> gpurun_out/bench_full.json
#   wl         bench.py --workload C2r C3 C4       -> gpurun_out/bench_<wl>.json
#   launches   ncu launch list of the bench        -> gpurun_out/launches.csv
#   ncu        ncu --set full of $NCU_K on tools/run_level.py --workload ${NCU_WL:-C2}
#   smoke      __graft_entry__.smoke()
#   cmd        eval "$CMD"
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
for s in "$@"; do
  echo "=== $s"
  case $s in
    tests) timeout 2400 python -m pytest tests -m gpu -x -q 2>&1 | tail -8 > gpurun_out/pytest_gpu.log; cat gpurun_out/pytest_gpu.log ;;
    tq) timeout 1800 python -m pytest tests -m gpu -x -q -k "$PYK" 2>&1 | tail -30 > gpurun_out/pytest_quick.log; cat gpurun_out/pytest_quick.log ;;
    bench) timeout 900 python bench.py --no-cpu-baseline $BENCH_ARGS > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err; tail -3 gpurun_out/bench_c2.err
           python tools/bench_brief.py gpurun_out/bench_c2.json ;;
    benchfull) timeout 1200 python bench.py $BENCH_ARGS > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err; tail -3 gpurun_out/bench_full.err
           python tools/bench_brief.py gpurun_out/bench_full.json ;;
    wl) for wl in ${WLS:-C2r C3 C4}; do
          timeout 900 python bench.py --workload $wl --no-cpu-baseline --no-e2e > gpurun_out/bench_$wl.json 2> gpurun_out/bench_$wl.err
          echo "== $wl rc=$?"; tail -2 gpurun_out/bench_$wl.err; python tools/bench_brief.py gpurun_out/bench_$wl.json
        done ;;
    launches) timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
                python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/b_ncu.log 2>&1
              python tools/launch_summary.py gpurun_out/launches.csv > gpurun_out/launches_summary.txt 2>&1; head -30 gpurun_out/launches_summary.txt ;;
    ncu) timeout 1500 ncu --set full --import-source on --clock-control none -k "regex:${NCU_K:-k_nbrscore}" \
              --launch-skip ${NCU_SKIP:-1} -c 1 -o gpurun_out/${NCU_OUT:-prof} python tools/run_level.py --workload ${NCU_WL:-C2} --steps 1 $NCU_ARGS \
              > gpurun_out/ncu_${NCU_OUT:-prof}.log 2>&1; tail -3 gpurun_out/ncu_${NCU_OUT:-prof}.log
         python tools/ncu_summary.py gpurun_out/${NCU_OUT:-prof}.ncu-rep > gpurun_out/${NCU_OUT:-prof}_summary.txt 2>&1; cat gpurun_out/${NCU_OUT:-prof}_summary.txt ;;
    smoke) timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke.log 2>&1; tail -2 gpurun_out/smoke.log ;;
    cmd) eval "$CMD" ;;
  esac
done
