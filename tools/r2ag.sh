timeout 900 python -m pytest tests/test_gpu_stream.py -x -q -k "pull or push" 2>&1 | tail -1
for n in 2 4; do
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2955$n tests/dist_check.py > gpurun_out/r2ag_dist$n.txt 2>&1; echo "dist$n rc=$?"; grep -E "PASS|FAIL|ghost|world=|Error" gpurun_out/r2ag_dist$n.txt | head -5
cmd="python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2959$n"
timeout 900 $cmd bench.py --gpus $n --steps 10 --warmup 3 --no-cpu-baseline --no-other-configs > gpurun_out/r2ag_bench$n.json 2> gpurun_out/r2ag_bench$n.err; echo "bench $n rc=$?"
python -c "
import json; d=json.loads(open('gpurun_out/r2ag_bench$n.json').read().strip().splitlines()[-1]); e=d['e2e']; print('$n solve ms', d['ms_per_step'], 'e2e ms', e['ms_per_step'], 'iters', d['config']['iterations'][:2])"
done
