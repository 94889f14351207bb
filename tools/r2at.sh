timeout 1200 python -m pytest tests/test_gpu_mesh.py tests/test_gpu_stencil.py tests/test_gpu_stream.py -x -q 2>&1 | tail -2
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r2at.json 2> gpurun_out/r2at.err; tail -2 gpurun_out/r2at.err
python -c "
import json; d=json.loads(open('gpurun_out/r2at.json').read().strip().splitlines()[-1]); print(d['ms_per_step'], json.dumps(d['other_configs']))"
