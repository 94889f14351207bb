timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29551 tests/dist_check.py > gpurun_out/r2u_dist4.txt 2>&1; echo "dist4 rc=$?"; grep -E "PASS|FAIL|stall|ghost push|world=" gpurun_out/r2u_dist4.txt | head
for n in 2 4; do
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2956$n bench.py --gpus $n --steps 10 --warmup 3 > gpurun_out/r2u_bench$n.json 2> gpurun_out/r2u_bench$n.err; echo "bench $n rc=$?"
python -c "
import json; d=json.loads(open('gpurun_out/r2u_bench$n.json').read().strip().splitlines()[-1]); print('$n solve ms', d['ms_per_step'], 'e2e ms', d['e2e']['ms_per_step'], 'iters', d['config']['iterations'][:2], 'value', d['value'])"
done
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29571 tools/mb_dist.py > gpurun_out/r2u_mbdist4.txt 2>&1; grep "world=" gpurun_out/r2u_mbdist4.txt
