for v in "$@"; do echo "variant $v"; AMRB_SWEEP_VARIANT=$v python scratch/mb_sweep.py 2>&1 | head -1; done
