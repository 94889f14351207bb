timeout 900 python -m pytest tests/test_gpu_stream.py -x -q -k "pull or push" 2>&1 | tail -3
timeout 1500 python -m pytest tests/test_gpu_mlmg.py tests/test_gpu_mlmg_headline.py -x -q 2>&1 | tail -3
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29551 tests/dist_check.py > gpurun_out/r2ae_dist2.txt 2>&1; echo "dist2 rc=$?"; grep -E "PASS|FAIL|stall|ghost|world=|Error" gpurun_out/r2ae_dist2.txt | head
for n in 1 2; do
if [ $n = 1 ]; then cmd="python"; else cmd="python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2959$n"; fi
timeout 900 $cmd bench.py --gpus $n --steps 10 --warmup 3 --no-cpu-baseline --no-other-configs > gpurun_out/r2ae_bench$n.json 2> gpurun_out/r2ae_bench$n.err; echo "bench $n rc=$?"
python -c "
import json; d=json.loads(open('gpurun_out/r2ae_bench$n.json').read().strip().splitlines()[-1]); e=d['e2e']; print('$n solve ms', d['ms_per_step'], 'e2e ms', e['ms_per_step'], 'iters', d['config']['iterations'][:2])"
done
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29571 tools/mb_dist.py 2>&1 | grep "world="
