timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29594 tools/mb_interfere.py 2>&1 | grep -E "world=|Error" | head -30
