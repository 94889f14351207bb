import sys, ctypes as C, torch
sys.path.insert(0, '/root/repo')
import paper_2009_12009_b200 as A
L = C.CDLL('/root/repo/scratch/librowcopy.so')
n, m = 256, 64
dom = A.Box((0,0,0),(n-1,)*3); ba = A.BoxArray([dom]).max_size(m)
dm = A.DistributionMapping.single_rank(len(ba))
for g in (2,):
    a = A.MultiFab(ba, dm, 1, g); b = A.MultiFab(ba, dm, 1, g)
    t = a.fabtab
    bstride = int(t[1,0]-t[0,0]); pitch=int(t[0,3]); E1=int(t[0,2]//t[0,3]); front=(4-g%4)%4
    st = torch.cuda.current_stream().cuda_stream
    def run(grid, block, rpw, sc):
        L.launch_rowcopy(C.c_void_p(a.storage.data_ptr()), C.c_void_p(b.storage.data_ptr()), C.c_longlong(bstride), pitch, E1, g, front, 64, 64, rpw, grid, block, C.c_void_p(st), sc)
    for (grid, block, rpw, sc) in ((148*8, 256, 1, 0), (148*8, 256, 1, 1), (148*8, 256, 4, 1)):
        for _ in range(3): run(grid, block, rpw, sc)
        e0=torch.cuda.Event(enable_timing=True); e1=torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(20): run(grid, block, rpw, sc)
        e1.record(); torch.cuda.synchronize()
        us=e0.elapsed_time(e1)/20*1e3
        print(f"g={g} rowcopy scatter={sc} rpw={rpw}: {us:.1f} us  {2*n**3*8/us/1e3:.0f} GB/s")
N=a.storage.numel()
for _ in range(3): L.launch_flat(C.c_void_p(a.storage.data_ptr()), C.c_void_p(b.storage.data_ptr()), C.c_longlong(N), 148*8, 256, C.c_void_p(st))
e0=torch.cuda.Event(enable_timing=True); e1=torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(20): L.launch_flat(C.c_void_p(a.storage.data_ptr()), C.c_void_p(b.storage.data_ptr()), C.c_longlong(N), 148*8, 256, C.c_void_p(st))
e1.record(); torch.cuda.synchronize(); us=e0.elapsed_time(e1)/20*1e3
print(f"flat copy {N*8/1e6:.0f}MB: {us:.1f} us {2*N*8/us/1e3:.0f} GB/s")
