timeout 900 python -m pytest tests/test_gpu_mlmg.py tests/test_gpu_mlmg_headline.py -x -q 2>&1 | tail -1
for r in 1 2; do
timeout 900 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-other-configs > gpurun_out/r2as.json 2> gpurun_out/r2as.err
python -c "
import json; d=json.loads(open('gpurun_out/r2as.json').read().strip().splitlines()[-1]); print(d['ms_per_step'], d['e2e']['ms_per_step'], d['config']['oracle_parity'])"
done
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29871 tools/mb_dist.py 2>&1 | grep -E "grid|iteration"
