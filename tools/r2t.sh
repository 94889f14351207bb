timeout 2400 python -m pytest tests -q -m gpu 2>&1 | tail -3
python tools/mb_cycle_list.py > gpurun_out/plain.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/r2t_cycle.csv python tools/mb_cycle_list.py > gpurun_out/r2t_ncu.log 2>&1; tail -1 gpurun_out/r2t_ncu.log
