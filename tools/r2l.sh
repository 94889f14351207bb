timeout 900 python -m pytest tests/test_gpu_stream.py -x -q 2>&1 | tail -3
MB_CONFIGS=0,1,2,4 MB_CASES=256/256,128/128 timeout 600 python tools/mb_stream.py 2>&1 | grep -v legacy | tail -40
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2l_bench.json 2> gpurun_out/r2l_bench.err; python -c "
import json; d=json.loads(open('gpurun_out/r2l_bench.json').read().strip().splitlines()[-1]); print('solve ms', d['ms_per_step'], 'e2e ms', d['e2e']['ms_per_step'], 'iters', d['config']['iterations'][:2], 'frac', d['roofline']['frac'])"; tail -3 gpurun_out/r2l_bench.err
