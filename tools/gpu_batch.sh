cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --share-device --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_2rank.json 2> gpurun_out/bench_2rank.err; echo "2rank rc=$?"; grep -E "Error" gpurun_out/bench_2rank.err | head -3
python tools/bench_brief.py gpurun_out/bench_2rank.json; python -c "
import json; d=json.loads(open('gpurun_out/bench_2rank.json').read().strip().splitlines()[-1]); print(d['level'].get('phase_ms')); print(d.get('hierarchy')); print(d['config']['parallelism'])"
