CUDA_VISIBLE_DEVICES=0 timeout 900 python -m pytest tests/test_gpu_mlmg.py -x -q > gpurun_out/r1g_cl2_mlmg.log 2>&1; echo "rc=$?" >> gpurun_out/r1g_cl2_mlmg.log
AMRB_CLUSTER_TAIL=2 CUDA_VISIBLE_DEVICES=0 timeout 900 python -m pytest tests/test_gpu_mlmg.py -x -q -k "noncubic or cluster" > gpurun_out/r1g_cl2_mlmg_opt.log 2>&1; echo "rc=$?" >> gpurun_out/r1g_cl2_mlmg_opt.log
tail -2 gpurun_out/r1g_cl2_mlmg.log gpurun_out/r1g_cl2_mlmg_opt.log
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29622 tests/dist_check.py > gpurun_out/r1g_cl2_dist2.log 2>&1; echo "dist2 rc=$?"; grep "PASS\|FAIL" gpurun_out/r1g_cl2_dist2.log
python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29632 bench.py --gpus 2 > gpurun_out/r1g_cl2_n2.json 2> gpurun_out/r1g_cl2_n2.err
python -c "import json,sys;d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]);print(sys.argv[1],d['value'],d['ms_per_step'])" gpurun_out/r1g_cl2_n2.json
python -c "import __graft_entry__ as g; g.smoke(); print('SMOKE OK')" 2>&1 | tail -2
