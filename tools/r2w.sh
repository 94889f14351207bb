set -x
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29531 tests/dist_check.py > gpurun_out/r2w_dist2.txt 2>&1; echo "dist_check rc=$?"; grep -E "PASS|FAIL|Error|stall|ghost|world=" gpurun_out/r2w_dist2.txt | head -12
for gp in auto off; do
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29532 bench.py --gpus 2 --steps 10 --warmup 3 --no-cpu-baseline --no-other-configs --ghost-push $gp > gpurun_out/r2w_bench2_$gp.json 2> gpurun_out/r2w_bench2_$gp.err; echo "bench $gp rc=$?"
python -c "
import json; d=json.loads(open('gpurun_out/r2w_bench2_$gp.json').read().strip().splitlines()[-1]); print('$gp solve ms', d['ms_per_step'], 'e2e ms', d['e2e']['ms_per_step'], 'iters', d['config']['iterations'][:2])"
done
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29571 tools/mb_dist.py > gpurun_out/r2w_mbdist2.txt 2>&1; grep -v Warn gpurun_out/r2w_mbdist2.txt | tail -40
