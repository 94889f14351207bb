for d in "$@"; do echo "dbg $d"; AMRB_SWEEP_VARIANT=11 AMRB_DBG=$d python scratch/mb_sweep.py 2>&1 | head -1; done
