for v in 2 6 10 14; do for c in 4 8 16; do echo "variant $v chunk $c"; AMRB_SWEEP_CHUNK=$c AMRB_SWEEP4_VARIANT=$v python scratch/mb_sweep.py 2>&1 | head -1; done; done
