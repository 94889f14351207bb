timeout 1500 python -m pytest tests/test_gpu_mlmg.py tests/test_gpu_mlmg_headline.py -x -q 2>&1 | tail -1
for n in 1 2 4; do
if [ $n = 1 ]; then cmd="python"; else cmd="python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2979$n"; fi
timeout 900 $cmd bench.py --gpus $n --steps 10 --warmup 3 --no-cpu-baseline --no-other-configs > gpurun_out/r2ak_bench$n.json 2> gpurun_out/r2ak_bench$n.err; echo "bench $n rc=$?"
python -c "
import json; d=json.loads(open('gpurun_out/r2ak_bench$n.json').read().strip().splitlines()[-1]); e=d['e2e']; print('$n solve ms', d['ms_per_step'], 'e2e ms', e['ms_per_step'], 'iters', d['config']['iterations'][:2])"
done
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29741 tests/dist_check.py > gpurun_out/r2ak_dist4.txt 2>&1; echo "dist4 rc=$?"; grep -E "PASS|FAIL" gpurun_out/r2ak_dist4.txt | head -3
