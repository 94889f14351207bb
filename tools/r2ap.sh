for rep in 1 2; do for p in 2 1; do
timeout 900 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-other-configs --option pdl=$p > gpurun_out/r2ap.json 2> gpurun_out/r2ap.err
python -c "
import json; d=json.loads(open('gpurun_out/r2ap.json').read().strip().splitlines()[-1]); e=d['e2e']; print('pdl=$p solve ms %.3f e2e ms %.3f' % (d['ms_per_step'], e['ms_per_step']))"
done; done
