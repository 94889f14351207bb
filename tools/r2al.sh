for rep in 1 2; do
for v in "off" "remote" "remote --option push_fence=1" "on"; do
for n in 2 4; do
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2980$n bench.py --gpus $n --steps 10 --warmup 3 --no-cpu-baseline --no-other-configs --ghost-push $v > gpurun_out/r2al.json 2> gpurun_out/r2al.err || tail -3 gpurun_out/r2al.err
python -c "
import json; d=json.loads(open('gpurun_out/r2al.json').read().strip().splitlines()[-1]); e=d['e2e']; print('$n GPUs push=$v solve ms %.3f e2e ms %.3f' % (d['ms_per_step'], e['ms_per_step']))"
done; done; done
