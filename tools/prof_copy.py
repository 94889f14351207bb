"""ncu target: the layout copy around a C3 solve (64 boxes of 64^3, ghost 1 ->
one 256^3 box, ghost 2), as MLMG.set_phi runs it."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2009_12009_b200 as A
dom = A.Box((0, 0, 0), (255, 255, 255))
ba = A.BoxArray([dom]).max_size(64)
dm = A.DistributionMapping.single_rank(len(ba))
tr = A.Transport(1)
src = A.MultiFab(ba, dm, 1, 1)
dst = A.MultiFab(A.BoxArray([dom]), A.DistributionMapping.single_rank(1), 1, 2)
src.storage.normal_()
for _ in range(4):
    A.parallel_copy(dst, src, tr)
torch.cuda.synchronize()
