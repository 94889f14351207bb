CUDA_VISIBLE_DEVICES=0 timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/r1g_final_gputests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r1g_final_gputests.log
CUDA_VISIBLE_DEVICES=0 python -c "import __graft_entry__ as g; g.smoke(); print('SMOKE OK')" > gpurun_out/r1g_final_smoke.log 2>&1
for n in 2 4; do
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2971$n tests/dist_check.py > gpurun_out/r1g_final_dist$n.log 2>&1; echo "dist$n rc=$?" >> gpurun_out/r1g_final_smoke.log
done
CUDA_VISIBLE_DEVICES=0 python bench.py > gpurun_out/r1g_final_bench.json 2> gpurun_out/r1g_final_bench.err
CUDA_VISIBLE_DEVICES=0 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r1g_final_ref.json 2> gpurun_out/r1g_final_ref.err
for n in 2 4; do
python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2973$n bench.py --gpus $n > gpurun_out/r1g_final_n$n.json 2> gpurun_out/r1g_final_n$n.err
done
tail -n 3 gpurun_out/r1g_final_gputests.log; cat gpurun_out/r1g_final_smoke.log | tail -n 4; grep PASS gpurun_out/r1g_final_dist*.log
for f in gpurun_out/r1g_final_bench.json gpurun_out/r1g_final_ref.json gpurun_out/r1g_final_n2.json gpurun_out/r1g_final_n4.json; do python -c "import json,sys;d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]);print(sys.argv[1],d['value'],d['ms_per_step'],d.get('e2e',{}).get('ms_per_step'),d.get('roofline',{}).get('frac'),d.get('clocks',{}).get('reasons'))" $f; done
