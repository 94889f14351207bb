timeout 900 python bench.py --config c5 --steps 5 --warmup 3 > gpurun_out/r2av.json 2> gpurun_out/r2av.err; echo rc=$?; tail -2 gpurun_out/r2av.err
python -c "
import json; d=json.loads(open('gpurun_out/r2av.json').read().strip().splitlines()[-1]); print(d['metric'][:60], d['value'], d['ms_per_step'], d['e2e']['ms_per_step'], d['roofline']['frac'], (d.get('cpu_baseline') or {}).get('value'))"
