set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 2700 python -m pytest tests -q -m gpu 2>&1 | tail -3
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
CUDA_VISIBLE_DEVICES=0 timeout 900 python bench.py > gpurun_out/r2f_bench.json 2> gpurun_out/r2f_bench.err; echo "bench rc=$?"
CUDA_VISIBLE_DEVICES=0 timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r2f_ref.json 2> gpurun_out/r2f_ref.err; echo "ref rc=$?"
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29731 tests/dist_check.py > gpurun_out/r2f_dist2.txt 2>&1; echo "dist2 rc=$?"
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29732 bench.py --gpus 2 > gpurun_out/r2f_n2.json 2> gpurun_out/r2f_n2.err; echo "n2 rc=$?"
CUDA_VISIBLE_DEVICES=0 python tools/mb_cycle_list.py > gpurun_out/plain.log 2>&1 && CUDA_VISIBLE_DEVICES=0 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/r2f_cycle.csv python tools/mb_cycle_list.py > gpurun_out/r2f_ncu.log 2>&1; tail -1 gpurun_out/r2f_ncu.log
CUDA_VISIBLE_DEVICES=0 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2f_bench_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-other-configs > gpurun_out/r2f_ncu_bench.log 2>&1; tail -1 gpurun_out/r2f_ncu_bench.log
CUDA_VISIBLE_DEVICES=0 python profiles/prof_fine_sweep.py > gpurun_out/plain.log 2>&1 && CUDA_VISIBLE_DEVICES=0 ncu --set full --clock-control none --import-source on -k regex:k_gsrb_stream -s 4 -c 1 -o gpurun_out/r2f_fine -f python profiles/prof_fine_sweep.py > gpurun_out/r2f_ncu_full.log 2>&1; tail -1 gpurun_out/r2f_ncu_full.log
for f in gpurun_out/r2f_bench.json gpurun_out/r2f_ref.json gpurun_out/r2f_n2.json; do python -c "import json,sys;d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]);print(sys.argv[1],d['value'],d['ms_per_step'],d.get('e2e',{}).get('ms_per_step'),d.get('roofline',{}).get('frac'),d.get('clocks',{}).get('reasons'))" $f; done
grep -E "PASS|FAIL|ghost|world=" gpurun_out/r2f_dist2.txt | head
