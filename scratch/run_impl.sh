for v in 4 5; do echo "impl $v t16=32"; AMRB_SWEEP_T16=32 AMRB_SWEEP_IMPL=$v python scratch/mb_sweep.py 2>&1; done
