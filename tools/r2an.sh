timeout 2700 python -m pytest tests -q -m gpu -x 2>&1 | tail -2
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29741 tests/dist_check.py > gpurun_out/r2an_dist4.txt 2>&1; echo "dist4 rc=$?"; grep -E "PASS|FAIL|ghost" gpurun_out/r2an_dist4.txt | head -5
for n in 1 2 4; do
if [ $n = 1 ]; then cmd="python"; else cmd="python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2981$n"; fi
timeout 900 $cmd bench.py --gpus $n --steps 10 --warmup 3 --no-cpu-baseline --no-other-configs > gpurun_out/r2an_bench$n.json 2> gpurun_out/r2an_bench$n.err; echo "bench $n rc=$?"
python -c "
import json; d=json.loads(open('gpurun_out/r2an_bench$n.json').read().strip().splitlines()[-1]); e=d['e2e']; print('$n solve ms %.3f e2e ms %.3f' % (d['ms_per_step'], e['ms_per_step']), d['config']['iterations'][:2])"
done
