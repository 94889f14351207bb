for cl in 1 2; do for gr in default 0; do
if [ $gr = default ]; then unset MB_GRID; else export MB_GRID=$gr; fi
echo "cluster=$cl grid=$gr"
MB_CLUSTER=$cl timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 2978$cl tools/mb_dist.py 2>&1 | grep -E "levels:|level_grid|coarse tail|iteration"
done; done
