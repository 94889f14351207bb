CUDA_VISIBLE_DEVICES=0 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r1g_ref_mt.json 2> gpurun_out/r1g_ref_mt.err
CUDA_VISIBLE_DEVICES=0 python bench.py > gpurun_out/r1g_n1.json 2> gpurun_out/r1g_n1.err
for n in 2 4; do
python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus $n > gpurun_out/r1g_n$n.json 2> gpurun_out/r1g_n$n.err
done
for f in gpurun_out/r1g_ref_mt.json gpurun_out/r1g_n1.json gpurun_out/r1g_n2.json gpurun_out/r1g_n4.json; do python -c "import json,sys;d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]);print(sys.argv[1],d['value'],d['ms_per_step'],d.get('cpu_baseline',{}).get('value'),d.get('clocks'))" $f; done
