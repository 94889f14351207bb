for v in 0 1; do echo "align $v"; AMRB_SWEEP_ALIGN=$v python scratch/mb_sweep.py 2>&1; done
