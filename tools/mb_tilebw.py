# build first: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -shared -Xcompiler -fPIC -lcuda tools/tilebw.cu -o tools/libtilebw.so
import ctypes as C
L = C.CDLL('/root/repo/tools/libtilebw.so')
us = C.c_float()
for rows in (20, 36):
    for mode, name in ((0, "ldg->sts"), (1, "cp.async16"), (2, "tma2d")):
        for st in ((2, 4) if mode < 2 else (2, 4, 8)):
            for cps in (1, 2):
                err = L.run_tilebw(mode, st, rows, cps, C.byref(us))
                nbytes = 256 * 128 * rows * 68 * 8
                print(f"rows={rows} {name:10s} stages={st} ctas/sm={cps}: {us.value:8.1f} us  {nbytes/us.value/1e3:7.0f} GB/s  err={err}", flush=True)
