for n in 1 2; do
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2952$n tools/mb_dist.py > gpurun_out/r2n_dist_n$n.txt 2>&1
done
cat gpurun_out/r2n_dist_n*.txt | grep -v Warning | grep -E "world=|levels|Error|error" | tail -60
