nvidia-smi topo -m 2>&1 | head -20
lscpu | grep -iE "numa|socket|model name|^cpu\(s\)"
for n in 1 4; do for b in nobind bind; do
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2958$n tools/mb_h2d.py $b 2>&1 | grep world=
done; done
