timeout 900 python -m pytest tests/test_gpu_mlmg.py tests/test_gpu_mlmg_headline.py -x -q 2>&1 | tail -2
for r in 1 2; do
timeout 900 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-other-configs > gpurun_out/r2aw.json 2> gpurun_out/r2aw.err; tail -1 gpurun_out/r2aw.err
python -c "
import json; d=json.loads(open('gpurun_out/r2aw.json').read().strip().splitlines()[-1]); e=d['e2e']; print('solve ms', d['ms_per_step'], 'e2e ms', e['ms_per_step'], e['serial']['ms_per_step'], e['bounds'], d['config']['iterations'][:3], d['config']['oracle_parity']['history_equals_oracle'], d['config']['oracle_parity']['phi_sha256_equals_oracle'])"
done
for n in 2 4; do
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2991$n bench.py --gpus $n --steps 20 --warmup 5 --no-cpu-baseline --no-other-configs > gpurun_out/r2aw_n$n.json 2> gpurun_out/r2aw_n$n.err
python -c "
import json; d=json.loads(open('gpurun_out/r2aw_n$n.json').read().strip().splitlines()[-1]); e=d['e2e']; print('$n solve ms', d['ms_per_step'], 'e2e ms', e['ms_per_step'], d['config']['iterations'][:3])"
done
