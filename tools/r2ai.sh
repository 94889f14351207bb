timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29741 tests/dist_check.py > gpurun_out/r2ai_dist4.txt 2>&1; echo "dist4 rc=$?"; grep -E "PASS|FAIL|ghost|world=|stall" gpurun_out/r2ai_dist4.txt | head
for n in 2 4; do
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2975$n bench.py --gpus $n > gpurun_out/r2ai_n$n.json 2> gpurun_out/r2ai_n$n.err; echo "n$n rc=$?"
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2976$n bench.py --impl reference --gpus $n --steps 3 --warmup 3 > gpurun_out/r2ai_ref_n$n.json 2> gpurun_out/r2ai_ref_n$n.err; echo "ref n$n rc=$?"
done
for f in gpurun_out/r2ai_n2.json gpurun_out/r2ai_n4.json gpurun_out/r2ai_ref_n2.json gpurun_out/r2ai_ref_n4.json; do python -c "import json,sys;d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]);print(sys.argv[1],d['value'],d['ms_per_step'],d.get('e2e',{}).get('ms_per_step'),d.get('roofline',{}).get('frac'),d.get('clocks',{}).get('reasons'))" $f; done
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29771 tools/mb_dist.py 2>&1 | grep "world=" > gpurun_out/r2ai_mbdist4.txt; cat gpurun_out/r2ai_mbdist4.txt
