export MB_CFGS=128/128,64/64
echo "sweep5 16x64"; python scratch/mb_sweep.py
echo "sweep5 16x32"; AMRB_SWEEP_TK=32 python scratch/mb_sweep.py
echo "sweep4 (impl 4)"; AMRB_SWEEP_IMPL=4 python scratch/mb_sweep.py
