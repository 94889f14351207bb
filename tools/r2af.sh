python tools/mb_pull.py
python tools/mb_pull.py prof > /dev/null 2>&1 && ncu --set full --clock-control none --import-source on -k regex:k_gsrb_stream -s 2 -c 1 -o gpurun_out/r2af_pull -f python tools/mb_pull.py prof > gpurun_out/r2af_ncu.log 2>&1; tail -2 gpurun_out/r2af_ncu.log
