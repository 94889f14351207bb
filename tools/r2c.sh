timeout 600 python -m pytest tests/test_gpu_stream.py -x -q 2>&1 | tail -15
timeout 300 python tools/mb_stream.py 2>&1 | tail -30
python tools/prof_stream.py sweep > gpurun_out/plain.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:k_gsrb_stream -s 3 -c 1 -o gpurun_out/r2c_stream -f python tools/prof_stream.py sweep > gpurun_out/r2c_ncu.log 2>&1
tail -3 gpurun_out/r2c_ncu.log
