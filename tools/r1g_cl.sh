export CUDA_VISIBLE_DEVICES_ALL=$CUDA_VISIBLE_DEVICES
CUDA_VISIBLE_DEVICES=0 timeout 900 python -m pytest tests/test_gpu_mlmg.py -x -q > gpurun_out/r1g_cl_mlmg.log 2>&1; echo "rc=$?" >> gpurun_out/r1g_cl_mlmg.log
tail -3 gpurun_out/r1g_cl_mlmg.log
for n in 2 4; do
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2961$n tests/dist_check.py > gpurun_out/r1g_cl_dist$n.log 2>&1; echo "dist$n rc=$?"; grep -v "Warning\|frame\|^\*\|OMP\|Symmetric\|CUDA driver\|Exception raised" gpurun_out/r1g_cl_dist$n.log | tail -4
done
CUDA_VISIBLE_DEVICES=0 python bench.py --no-cpu-baseline > gpurun_out/r1g_cl_n1.json 2> gpurun_out/r1g_cl_n1.err
for n in 2 4; do
python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2953$n bench.py --gpus $n > gpurun_out/r1g_cl_n$n.json 2> gpurun_out/r1g_cl_n$n.err
AMRB_CLUSTER_TAIL=0 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2954$n bench.py --gpus $n > gpurun_out/r1g_nocl_n$n.json 2> gpurun_out/r1g_nocl_n$n.err
done
for f in gpurun_out/r1g_cl_n1.json gpurun_out/r1g_cl_n2.json gpurun_out/r1g_nocl_n2.json gpurun_out/r1g_cl_n4.json gpurun_out/r1g_nocl_n4.json; do python -c "import json,sys;d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]);print(sys.argv[1],d['value'],d['ms_per_step'],d['config'].get('iterations',[None])[:2],d.get('clocks',{}).get('reasons'))" $f; done
