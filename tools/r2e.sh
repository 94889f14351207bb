timeout 1500 python -m pytest tests -x -q -m gpu 2>&1 | tail -5
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2e_bench.json 2> gpurun_out/r2e_bench.err; tail -c 2500 gpurun_out/r2e_bench.json
python profiles/prof_fine_sweep.py > gpurun_out/plain.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:k_gsrb_stream -s 4 -c 1 -o gpurun_out/r2e_fine -f python profiles/prof_fine_sweep.py > gpurun_out/r2e_ncu.log 2>&1; tail -2 gpurun_out/r2e_ncu.log
