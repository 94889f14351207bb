timeout 600 python -m pytest tests/test_gpu_stream.py -x -q 2>&1 | tail -30
timeout 300 python tools/mb_stream.py 2>&1 | tail -30
