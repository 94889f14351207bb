set -x
python -m pytest tests -m gpu -x -q > gpurun_out/r1g_gputests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r1g_gputests.log
python -c "import __graft_entry__ as g; g.smoke(); print('SMOKE OK')" > gpurun_out/r1g_smoke.log 2>&1
python bench.py > gpurun_out/r1g_bench.json 2> gpurun_out/r1g_bench.err
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r1g_ref.json 2> gpurun_out/r1g_ref.err
tail -3 gpurun_out/r1g_gputests.log; cat gpurun_out/r1g_smoke.log | tail -2; cat gpurun_out/r1g_bench.json | head -c 400
