timeout 900 python -m pytest tests/test_gpu_mlmg.py tests/test_gpu_mlmg_headline.py -x -q -k "external or boundary or dirichlet" 2>&1 | tail -15
