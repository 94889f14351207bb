timeout 900 python -m pytest tests/test_gpu_mesh.py -x -q 2>&1 | tail -2
timeout 1500 python -m pytest tests/test_gpu_mlmg.py tests/test_gpu_mlmg_headline.py tests/test_gpu_stream.py -x -q 2>&1 | tail -2
for r in 1 2; do
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-other-configs > gpurun_out/r2am_bench.json 2> gpurun_out/r2am_bench.err; echo "bench rc=$?"
python -c "
import json; d=json.loads(open('gpurun_out/r2am_bench.json').read().strip().splitlines()[-1]); e=d['e2e']; print('solve ms', d['ms_per_step'], 'e2e ms', e['ms_per_step'], 'iters', d['config']['iterations'][:2], 'frac', d['roofline']['frac'])"
done
python tools/mb_cycle_list.py > gpurun_out/plain.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/r2am_cycle.csv python tools/mb_cycle_list.py > gpurun_out/r2am_ncu.log 2>&1; tail -1 gpurun_out/r2am_ncu.log
