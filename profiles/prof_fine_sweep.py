"""Launch the bench's roofline kernel alone for ncu: the C3 solver's internal
level-0 layout (one 256^3 box, phi grown by 2, rhs by 1), fill + fused GSRB
sweep, 12 times.  Only the sweeps launch k_gsrb_stream, so

    ncu --set full --clock-control none -k regex:k_gsrb_stream -s 4 -c 1 \\
        -o gpurun_out/fine_sweep python profiles/prof_fine_sweep.py

captures a warm fine-level launch; `python profiles/prof_fine_sweep.py --summarize
rep.ncu-rep` writes profiles/fine_sweep_traffic.json (dram bytes per launch),
which bench.py reports as roofline.traffic."""

import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def run():
    import torch

    import paper_2009_12009_b200 as A
    from paper_2009_12009_b200 import stencil as S

    dom = A.Box((0, 0, 0), (255, 255, 255))
    ba = A.BoxArray([dom]).max_size(64)
    dm = A.DistributionMapping.single_rank(len(ba))
    tr = A.Transport(1)
    geom = A.Geometry(dom, (0.0,) * 3, (1.0,) * 3, True)
    mg = A.MLMG(geom, ba, dm, transport=tr)
    top = mg.levels[0]
    a, b = top.phi[0], top.phi[1]
    a.storage.normal_()
    top.rhs.storage.normal_()
    for _ in range(12):
        A.fill_boundary(a, tr, top.domain, True, ngrow=2)
        S.gsrb_sweep(a, b, top.rhs, top.dh)
        a, b = b, a
    torch.cuda.synchronize()
    print("layout:", [tuple(top.ba[i].extents()) for i in range(len(top.ba))])


def summarize(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    import csv
    import io

    rows = list(csv.reader(io.StringIO(out)))
    h, u, v = rows[0], rows[1], rows[2]
    get = {a: (b, c) for a, b, c in zip(h, u, v)}

    def mb(key):
        unit, val = get[key]
        scale = {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3}[unit]
        return float(val) * scale

    res = {
        "kernel": get["Kernel Name"][1] if "Kernel Name" in get else "k_gsrb_stream",
        "layout": "C3 solver level 0: one 256^3 box, phi ngrow 2, rhs ngrow 1",
        "dram_read_mb": mb("dram__bytes_read.sum"),
        "dram_write_mb": mb("dram__bytes_write.sum"),
        "duration_us": float(get["gpu__time_duration.sum"][1]),
        "source": os.path.basename(rep) + " (ncu --set full --clock-control none)",
        "alg_bytes_per_launch": 24 * 256**3 + 8 * 6 * 256**2,
    }
    res["traffic_bytes_per_launch"] = int(round((res["dram_read_mb"] + res["dram_write_mb"]) * 1e6))
    with open(os.path.join(ROOT, "profiles", "fine_sweep_traffic.json"), "w") as f:
        json.dump(res, f, indent=1)
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    if len(sys.argv) > 2 and sys.argv[1] == "--summarize":
        summarize(sys.argv[2])
    else:
        run()
