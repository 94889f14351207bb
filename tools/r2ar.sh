timeout 900 python -m pytest tests/test_gpu_mlmg.py tests/test_gpu_mlmg_headline.py -x -q 2>&1 | tail -2
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-other-configs > gpurun_out/r2ar.json 2> gpurun_out/r2ar.err
python -c "
import json; d=json.loads(open('gpurun_out/r2ar.json').read().strip().splitlines()[-1]); print(d['ms_per_step'], d['config']['iterations'], d['config']['oracle_parity'])"
