echo "sweep5 16x64 (default)"; python tools/mb_level1.py
echo "sweep5 16x32"; AMRB_SWEEP_TK=32 python tools/mb_level1.py
echo "sweep4"; AMRB_SWEEP_IMPL=4 python tools/mb_level1.py
