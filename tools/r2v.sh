timeout 900 python -m pytest tests/test_gpu_mlmg.py -x -q -k "grid or cluster or noncubic" 2>&1 | tail -2
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29541 tools/mb_dist.py 2>&1 | grep -i "grid\|iteration\|tail"
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29542 tools/mb_dist.py 2>&1 | grep -i "grid\|iteration\|tail"
