set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 2700 python -m pytest tests -q -m gpu 2>&1 | tail -3
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
CUDA_VISIBLE_DEVICES=0 timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/r2i_bench.json 2> gpurun_out/r2i_bench.err; echo "bench rc=$?"
CUDA_VISIBLE_DEVICES=0 timeout 900 python bench.py --impl reference --gpus 1 --steps 3 --warmup 3 > gpurun_out/r2i_ref.json 2> gpurun_out/r2i_ref.err; echo "ref rc=$?"
for n in 2 4; do
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2983$n tests/dist_check.py > gpurun_out/r2i_dist$n.txt 2>&1; echo "dist$n rc=$?"
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2984$n bench.py --gpus $n --steps 20 --warmup 5 > gpurun_out/r2i_n$n.json 2> gpurun_out/r2i_n$n.err; echo "n$n rc=$?"
done
CUDA_VISIBLE_DEVICES=0 python tools/mb_cycle_list.py > gpurun_out/plain.log 2>&1 && CUDA_VISIBLE_DEVICES=0 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/r2i_cycle.csv python tools/mb_cycle_list.py > gpurun_out/r2i_ncu.log 2>&1; tail -1 gpurun_out/r2i_ncu.log
CUDA_VISIBLE_DEVICES=0 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2i_bench_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-other-configs > gpurun_out/r2i_ncu_bench.log 2>&1; tail -1 gpurun_out/r2i_ncu_bench.log
for f in gpurun_out/r2i_bench.json gpurun_out/r2i_ref.json gpurun_out/r2i_n2.json gpurun_out/r2i_n4.json; do python -c "import json,sys;d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]);print(sys.argv[1],d['value'],d['ms_per_step'],d.get('e2e',{}).get('ms_per_step'),d.get('roofline',{}).get('frac'),d.get('clocks',{}).get('reasons'))" $f; done
grep -E "PASS|FAIL" gpurun_out/r2i_dist*.txt
