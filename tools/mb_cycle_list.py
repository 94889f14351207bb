"""Two eager solve iterations of the C3 MLMG (one V-cycle + the fused norm
each) between cudaProfilerStart/Stop, for the ncu launch list:

    ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off \\
        --csv --log-file gpurun_out/cycle.csv python tools/mb_cycle_list.py
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2009_12009_b200 as A  # noqa: E402

dom = A.Box((0, 0, 0), (255, 255, 255))
ba = A.BoxArray([dom]).max_size(64)
dm = A.DistributionMapping.single_rank(len(ba))
tr = A.Transport(1)
geom = A.Geometry(dom, (0.0,) * 3, (1.0,) * 3, True)
mg = A.MLMG(geom, ba, dm, transport=tr, use_graph=False)
for lv in mg.levels:
    for f in lv.phi:
        f.storage.normal_()
    lv.rhs.storage.normal_()
mg._prime()
mg._body()
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
for _ in range(2):
    mg._body()
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
print("lag", mg.lag)
