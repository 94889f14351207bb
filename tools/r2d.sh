timeout 600 python -m pytest tests/test_gpu_stream.py -x -q 2>&1 | tail -3
MB_CONFIGS=0,1,2,3,4,5 timeout 600 python tools/mb_stream.py 2>&1 | grep -v legacy | tail -80
