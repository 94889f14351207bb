export MB_CFGS=256/256,512/128,512/512
echo "default (auto)"; python tools/mb_sweep.py
echo "forced 16x64"; AMRB_SWEEP_TK=64 python tools/mb_sweep.py
