AMRB_LIBRARY=checked timeout 600 python tools/sanitize.py 2>&1 | tail -4
timeout 900 python -m pytest tests/test_gpu_checked.py tests/test_gpu_stream.py -x -q 2>&1 | tail -3
