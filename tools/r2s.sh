timeout 900 python -m pytest tests/test_gpu_stream.py -x -q -k resid 2>&1 | tail -3
timeout 1500 python -m pytest tests/test_gpu_mlmg.py tests/test_gpu_mlmg_headline.py -x -q 2>&1 | tail -2
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29541 tools/mb_dist.py 2>&1 | grep -i "resid\|iteration"
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-other-configs > gpurun_out/r2s_bench.json 2> gpurun_out/r2s_bench.err; python -c "
import json; d=json.loads(open('gpurun_out/r2s_bench.json').read().strip().splitlines()[-1]); print('solve ms', d['ms_per_step'], 'e2e ms', d['e2e']['ms_per_step'], 'iters', d['config']['iterations'][:2], 'frac', d['roofline']['frac'])"; tail -3 gpurun_out/r2s_bench.err
