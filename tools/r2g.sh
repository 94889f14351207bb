timeout 1500 python -m pytest tests/test_gpu_mlmg.py tests/test_gpu_mlmg_headline.py -x -q 2>&1 | tail -15
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2g_bench.json 2> gpurun_out/r2g_bench.err; tail -c 1500 gpurun_out/r2g_bench.json; tail -5 gpurun_out/r2g_bench.err
