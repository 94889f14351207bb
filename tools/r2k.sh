timeout 900 python -m pytest tests/test_gpu_stream.py -x -q 2>&1 | tail -3
MB_CONFIGS=0,6,7 MB_CASES=512/32,256/32 timeout 600 python tools/mb_stream.py 2>&1 | tail -30
