CUDA_VISIBLE_DEVICES=0 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2ao_bench_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-other-configs > gpurun_out/r2ao_ncu_bench.log 2>&1; tail -1 gpurun_out/r2ao_ncu_bench.log
python profiles/summarize_launches.py gpurun_out/r2ao_bench_launches.csv "x" | grep k_copy
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2ao_bench.json 2> gpurun_out/r2ao_bench.err
python -c "
import json; d=json.loads(open('gpurun_out/r2ao_bench.json').read().strip().splitlines()[-1]); e=d['e2e']; print('solve ms', d['ms_per_step'], 'e2e ms', e['ms_per_step'], json.dumps(d['other_configs'])[:700])"
