for n in 1 4; do
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2959$n tools/mb_interfere.py 2>&1 | grep -E "world=|Error|error" | head -20
done
