timeout 1200 python -m pytest tests/test_gpu_mesh.py tests/test_gpu_plotfile.py tests/test_gpu_amr.py -x -q 2>&1 | tail -1
python tools/prof_copy.py && ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_copy --csv python tools/prof_copy.py 2>/dev/null | grep k_copy | tail -2
for r in 1 2; do
timeout 900 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r2ay.json 2> gpurun_out/r2ay.err; tail -1 gpurun_out/r2ay.err
python -c "
import json; d=json.loads(open('gpurun_out/r2ay.json').read().strip().splitlines()[-1]); e=d['e2e']; print('solve ms', d['ms_per_step'], 'e2e ms', e['ms_per_step'], d['config']['oracle_parity']['phi_sha256_equals_oracle'], json.dumps(d['other_configs']['c5'])[:200], d['other_configs']['c1']['fill_us'])"
done
