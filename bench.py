"""Benchmark: MLMG Poisson solve (C3: 256^3, 64^3 boxes, 1 GPU; C4 weak scaling:
256^3 per GPU) through the package API, plus the fused GSRB kernel roofline.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

One step = one full MLMG solve to 1e-10 relative residual on a synthetic,
host-centred random rhs.  ``value`` = GSRB cell-updates (every smoother
relaxation of every cell on every level) per second over the K timed solves,
whole job (all GPUs).  ``ms_per_step`` is the MLMG solve time.  ``e2e`` is the
same metric through MLMG.solve with the rhs in pinned host memory and the
solution copied back to pinned host memory inside the timed region.
``roofline`` is the fine-level fused GSRB sweep kernel, timed with CUDA events
on its launch stream, against the measured HBM copy bandwidth.

``--impl reference`` times the CPU oracle (numpy restatement of the reference, per-box loops on all host threads;
the reference itself has no MLMG) on rank 0: one V-cycle of the same
problem per step.
"""

from __future__ import annotations

import argparse
import hashlib
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
from golden.make_mlmg_golden import headline_rhs  # noqa: E402  (the synthetic-input recipe, numpy only)

METRIC = "fp64 cell-updates/s (GSRB, %HBM roofline); MLMG 256^3 solve time @1/2/4/8 GPU"
UNIT = "cell-updates/s"


def _traffic(alg_bytes):
    """dram read+write bytes per launch of the roofline kernel from the committed
    ncu capture (profiles/fine_sweep_traffic.json, see profiles/prof_fine_sweep.py);
    None when absent or captured on another layout."""
    try:
        with open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles", "fine_sweep_traffic.json")) as f:
            t = json.load(f)
        if "k_gsrb_stream" in t.get("kernel", "") and t.get("alg_bytes_per_launch", alg_bytes) == alg_bytes:
            return t["traffic_bytes_per_launch"]
    except (OSError, ValueError, KeyError):
        pass
    return None


def _golden_iterations(case):
    with open(os.path.join(ROOT, "tests", "golden", "mlmg_golden.json")) as f:
        return json.load(f)[case]["iterations"]


def _golden(case):
    with open(os.path.join(ROOT, "tests", "golden", "mlmg_golden.json")) as f:
        return json.load(f)[case]


def _peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


def _domain_for(n_gpus):
    f = {1: (1, 1, 1), 2: (2, 1, 1), 4: (2, 2, 1), 8: (2, 2, 2)}.get(n_gpus)
    if f is None:
        raise SystemExit(f"unsupported --gpus {n_gpus} (1, 2, 4 or 8)")
    return tuple(256 * x for x in f)


class ClockSampler:
    """SM clock and throttle reasons sampled every ~2 ms through NVML on a
    background thread while the timed region runs (nvidia-smi's 100 ms minimum
    period would catch one or two samples of a ~50 ms region)."""

    NAMES = (("hw_slowdown", "nvmlClocksEventReasonHwSlowdown"),
             ("hw_thermal_slowdown", "nvmlClocksEventReasonHwThermalSlowdown"),
             ("sw_thermal_slowdown", "nvmlClocksEventReasonSwThermalSlowdown"),
             ("sw_power_cap", "nvmlClocksEventReasonSwPowerCap"))

    def __init__(self, index):
        self.index = index
        self.rows = []
        self.err = None
        self._stop = None

    def __enter__(self):
        import threading

        try:
            import pynvml as N

            N.nvmlInit()
            vis = os.environ.get("CUDA_VISIBLE_DEVICES")
            idx = int(vis.split(",")[self.index]) if vis and vis.split(",")[self.index].isdigit() else self.index
            h = N.nvmlDeviceGetHandleByIndex(idx)
            self._max = float(N.nvmlDeviceGetMaxClockInfo(h, N.NVML_CLOCK_SM))
            bits = [(n, getattr(N, attr)) for n, attr in self.NAMES]
        except Exception as e:  # no NVML: report unsampled
            self.err = repr(e)
            return self
        self._stop = threading.Event()

        def run():
            while not self._stop.is_set():
                try:
                    clk = float(N.nvmlDeviceGetClockInfo(h, N.NVML_CLOCK_SM))
                    rs = N.nvmlDeviceGetCurrentClocksEventReasons(h)
                    self.rows.append((clk, [n for n, bit in bits if rs & bit]))
                except Exception as e:
                    self.err = repr(e)
                    return
                self._stop.wait(0.002)

        self._t = threading.Thread(target=run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        if self._stop is not None:
            self._stop.set()
            self._t.join(timeout=5)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "error": self.err}
        reasons = sorted({n for _, rs in self.rows for n in rs})
        return {"sm_mhz": float(np.median([c for c, _ in self.rows])), "sm_max_mhz": self._max,
                "reasons": reasons, "samples": len(self.rows), "source": "nvml, 2 ms period"}


def run_reference(args):
    """CPU oracle (numpy, per-box loops on a pool of all host threads) on rank 0; one V-cycle per step."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from oracle import mlmg_ref as R

    n, m = 256, 64
    boxes = [((i, j, k), (i + m - 1, j + m - 1, k + m - 1)) for i in range(0, n, m) for j in range(0, n, m)
             for k in range(0, n, m)]
    rhs = headline_rhs(n, 2)
    threads = os.cpu_count() or 1
    s = R.OracleMLMG(((0, 0, 0), (n - 1,) * 3), boxes, threads=threads)
    times = []
    for step in range(args.warmup + args.steps):
        s.cell_updates = 0
        t0 = time.perf_counter()
        s.solve(rhs, max_cycles=1)
        dt = time.perf_counter() - t0
        if step >= args.warmup:
            times.append((dt, s.cell_updates))
    tot_t = sum(t for t, _ in times)
    tot_u = sum(u for _, u in times)
    v = tot_u / tot_t
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1e3 * tot_t / len(times), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": "C3 MLMG Poisson 256^3, 64^3 boxes, periodic; one V(2,2) cycle per step (CPU sample)",
                   "global_batch": 1, "seq_len": n ** 3, "parallelism": "cpu"},
        "cpu_baseline": {"value": v, "unit": UNIT, "cores": threads, "kind": "port",
                         "sample": "one full V(2,2) cycle of the C3 solve (7 levels, 32-sweep bottom) in the numpy "
                                   "oracle, per-box loops on %d threads" % threads},
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def cpu_baseline_sample():
    """Bounded oracle sample for the cpu_baseline key (one V-cycle of C3)."""
    from oracle import mlmg_ref as R

    n, m = 256, 64
    boxes = [((i, j, k), (i + m - 1, j + m - 1, k + m - 1)) for i in range(0, n, m) for j in range(0, n, m)
             for k in range(0, n, m)]
    rhs = headline_rhs(n, 2)
    threads = os.cpu_count() or 1
    s = R.OracleMLMG(((0, 0, 0), (n - 1,) * 3), boxes, threads=threads)
    t0 = time.perf_counter()
    s.solve(rhs, max_cycles=1)
    dt = time.perf_counter() - t0
    return {"value": s.cell_updates / dt, "unit": UNIT, "cores": threads, "kind": "port",
            "sample": f"one V(2,2) cycle of C3 in the numpy oracle ({dt:.1f} s, {s.cell_updates} cell-updates), "
                      f"per-box loops on {threads} threads"}


def run_ours(args):
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    import paper_2009_12009_b200 as A
    from paper_2009_12009_b200 import stencil as S
    from paper_2009_12009_b200._native import lib

    ext = _domain_for(world)
    dom = A.Box((0, 0, 0), tuple(e - 1 for e in ext))
    ba = A.BoxArray([dom]).max_size(64)
    dm = A.sfc_distribute(ba, A.default_costs(ba), world)
    tr = A.Transport.distributed() if world > 1 else A.Transport(1)
    # weak scaling: the physical domain grows with the grid so cells stay cubic
    # (dx = 1/256 in every direction at every GPU count)
    geom = A.Geometry(dom, (0.0,) * 3, tuple(e / 256.0 for e in ext), True)

    # synthetic rhs: SURVEY 8(d)'s recipe, the same numpy bits the reference arm
    # and the golden oracle solve (tests/golden/make_mlmg_golden.py): seeded
    # standard normals over the global domain, host-centred (C3 seed 2, C4 seed 3)
    rhs_np = headline_rhs(ext, 2 if world == 1 else 3)
    rhs = A.MultiFab(ba, dm, 1, 0)
    rhs.load_valid_from(dom, rhs_np)
    rhs_sha = hashlib.sha256(rhs_np.tobytes()).hexdigest()
    del rhs_np
    phi = A.MultiFab(ba, dm, 1, 1)
    mg = A.MLMG(geom, ba, dm, transport=tr, ghost_push={"auto": None, "on": True, "off": False, "remote": "remote"}[args.ghost_push])

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier(device_ids=[local])
        torch.cuda.synchronize()

    def maxover(x):
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return t.item()

    def one_solve():
        phi.setval(0.0)
        return mg.solve(phi, rhs, rtol=1e-10, max_iter=100)

    for _ in range(args.warmup):
        one_solve()
    iters = []
    launches0 = lib().amrb_launch_count()
    replays0 = mg.graph_replays
    barrier()
    clk = ClockSampler(local)
    clk.__enter__()
    st = torch.cuda.current_stream()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(st)
    # back-to-back solves: each is queued before the previous one's result is
    # read (MLMG.solve(wait=False) / finish()), so the device never waits for
    # the host between solves; every solve runs to its own convergence test
    for s_ in range(args.steps):
        phi.setval(0.0)
        mg.solve(phi, rhs, rtol=1e-10, max_iter=100, wait=False)
        if s_ >= 1:
            mg.finish()
            iters.append(mg.iterations)
    mg.finish()
    iters.append(mg.iterations)
    e1.record(st)
    barrier()
    clk.__exit__(None, None, None)
    t_dev = maxover(e0.elapsed_time(e1) / 1e3)
    # the last timed solve against the CPU oracle's solve of the same rhs bits
    # (tests/golden/mlmg_golden.json; C3 only -- outside the timed region)
    parity = None
    if world == 1:
        gold = _golden("c3")
        out = A.gather_global(phi, dom)
        parity = {
            "history_equals_oracle": [float(x).hex() for x in mg.history] == gold["history"],
            "phi_sha256_equals_oracle": hashlib.sha256(np.ascontiguousarray(out).tobytes()).hexdigest()
            == gold["phi_sha256"],
            "solves_checked": "the last of the timed solves (the same MLMG object solved every step)",
        }
    # eager launches (uploads, priming sweep, copies) + the captured iteration's
    # launches times the iterations the device loop ran
    launches = (lib().amrb_launch_count() - launches0) + sum(iters) * mg.launches_per_cycle
    # every level's smoother relaxations, counted once for the whole job (replicated
    # bottom levels run redundantly on every rank but are counted once)
    updates_job = mg.cell_updates_per_cycle * sum(iters)
    # plain (unfused) fine-level sweeps per solve: nu1 + nu2 per cycle, one of
    # them fused with the prolongation when the up-leg is fused
    fine_per_step = (mg.nu1 + mg.nu2 - (1 if mg.levels[0].fuse else 0)) * sum(iters) / len(iters)
    value = updates_job / t_dev
    ms = 1e3 * t_dev / args.steps

    # ---- e2e: pinned host rhs -> solve -> pinned host phi ------------------------
    # Every step copies its rhs in from pinned host memory and its solution out
    # to pinned host memory inside the timed region.  Serial: copy in, solve,
    # copy out.  Pipelined (reported as `e2e`): double-buffered device rhs / phi,
    # step s+1's upload and step s's download run on a copy stream while step
    # s's solve runs (PCIe is full duplex; the solve does not touch the buffers
    # being copied).
    # host data as FabArray images (FabArray.from_host_image / to_host_image:
    # one contiguous copy + one scatter/gather launch each way)
    dev_rhs = [A.MultiFab(ba, dm, 1, 0), A.MultiFab(ba, dm, 1, 0)]
    dev_phi = [phi, A.MultiFab(ba, dm, 1, 1)]
    mine = rhs.image_size()
    host_rhs = torch.empty(mine, dtype=torch.float64).pin_memory()
    rhs.to_host_image(host_rhs)
    torch.cuda.synchronize()
    host_phi = [torch.empty(mine, dtype=torch.float64).pin_memory() for _ in range(2)]
    h2d = host_rhs.numel() * 8
    d2h = host_phi[0].numel() * 8

    def upload(x):
        dev_rhs[x].from_host_image(host_rhs, torch.cuda.current_stream())

    def download(x):
        dev_phi[x].to_host_image(host_phi[x], torch.cuda.current_stream())

    # untimed: first use of both buffers builds their staging and copy programs
    for x in (0, 1):
        upload(x)
        dev_phi[x].setval(0.0)
        mg.solve(dev_phi[x], dev_rhs[x], rtol=1e-10, max_iter=100)
        download(x)
    torch.cuda.synchronize()
    e_iters = []
    barrier()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        upload(0)
        dev_phi[0].setval(0.0)
        mg.solve(dev_phi[0], dev_rhs[0], rtol=1e-10, max_iter=100)
        e_iters.append(mg.iterations)
        download(0)
        torch.cuda.synchronize()
    barrier()
    t_serial = maxover(time.perf_counter() - t0)

    cs = torch.cuda.Stream()  # uploads
    ds = torch.cuda.Stream()  # downloads (PCIe is full duplex)
    main = torch.cuda.current_stream()
    rhs_ready = [torch.cuda.Event(), torch.cuda.Event()]
    solved = [torch.cuda.Event(), torch.cuda.Event()]
    fetched = [torch.cuda.Event(), torch.cuda.Event()]
    p_iters = []
    barrier()
    t0 = time.perf_counter()
    with torch.cuda.stream(cs):
        upload(0)
    rhs_ready[0].record(cs)
    for s_ in range(args.steps):
        cur, nxt = s_ % 2, (s_ + 1) % 2
        if s_ + 1 < args.steps:
            if s_ >= 1:
                cs.wait_event(solved[nxt])  # step s-1 is done with dev_rhs[nxt]
            with torch.cuda.stream(cs):
                upload(nxt)
            rhs_ready[nxt].record(cs)
        main.wait_event(rhs_ready[cur])
        if s_ >= 2:
            main.wait_event(fetched[cur])  # step s-2's solution has left dev_phi[cur]
        dev_phi[cur].setval(0.0)
        mg.solve(dev_phi[cur], dev_rhs[cur], rtol=1e-10, max_iter=100, wait=False)
        solved[cur].record(main)
        ds.wait_event(solved[cur])
        with torch.cuda.stream(ds):
            download(cur)
        fetched[cur].record(ds)
        if s_ >= 1:  # step s-1's result, read while step s runs
            mg.finish()
            p_iters.append(mg.iterations)
    mg.finish()
    p_iters.append(mg.iterations)
    torch.cuda.synchronize()
    barrier()
    t_e2e = maxover(time.perf_counter() - t0)
    e2e_value = mg.cell_updates_per_cycle * sum(p_iters) / t_e2e
    e2e_serial = mg.cell_updates_per_cycle * sum(e_iters) / t_serial

    # what bounds the pipelined loop: the same copies alone (both directions at
    # once, every rank at once) and the same solves alone, host-timed
    barrier()
    t0 = time.perf_counter()
    for s_ in range(args.steps):
        with torch.cuda.stream(cs):
            upload(s_ % 2)
        with torch.cuda.stream(ds):
            download(s_ % 2)
        torch.cuda.synchronize()
    barrier()
    t_copies = maxover(time.perf_counter() - t0)
    barrier()
    t0 = time.perf_counter()
    for s_ in range(args.steps):
        dev_phi[0].setval(0.0)
        mg.solve(dev_phi[0], dev_rhs[0], rtol=1e-10, max_iter=100)
    torch.cuda.synchronize()
    barrier()
    t_solves = maxover(time.perf_counter() - t0)

    # ---- roofline: fine-level fused sweep, events on its launch stream ----------
    top = mg.levels[0]
    a, b = top.phi[0], top.phi[1]
    evs = []
    for r in range(23):
        A.fill_boundary(a, tr, top.domain, True, ngrow=2)
        s0 = torch.cuda.Event(enable_timing=True)
        s1 = torch.cuda.Event(enable_timing=True)
        s0.record(st)
        S.gsrb_sweep(a, b, top.rhs, top.dh)
        s1.record(st)
        evs.append((s0, s1))
        a, b = b, a
    torch.cuda.synchronize()
    t_sweep = float(np.mean([x.elapsed_time(y) for x, y in evs[3:]])) / 1e3
    t_sweep = maxover(t_sweep)
    # algorithmic bytes of the launch as issued: the solver's internal level-0
    # layout (one box per rank), N valid cells, F face-ghost cells
    iba, idm = top.ba, top.dm
    nloc = sum(iba[i].num_cells() for i in range(len(iba)) if idm[i] == rank)
    floc = sum(2 * (e[0] * e[1] + e[1] * e[2] + e[2] * e[0]) for e in (iba[i].extents() for i in range(len(iba)) if idm[i] == rank))
    alg_bytes = 24 * nloc + 8 * floc
    achieved = alg_bytes / t_sweep / 1e9
    peak, peak_kind = _peaks()
    traffic = _traffic(alg_bytes)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline_sample()
    others = None
    if world == 1 and not args.no_other_configs:
        others = {"c1": c1_micro(), "c5": c5_micro()}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {
                "workload": ("C3 MLMG Poisson 256^3, 64^3 boxes, 1 GPU" if world == 1 else
                             f"C4 weak-scaling MLMG Poisson {ext[0]}x{ext[1]}x{ext[2]} (256^3 per GPU), 64^3 boxes"),
                "domain": list(ext), "box": 64, "boxes": len(ba), "levels": len(mg.levels), "cycle": "V(2,2)",
                "bottom_sweeps": mg.bottom_sweeps, "rtol": 1e-10, "iterations": iters,
                "rhs": "np.random.default_rng(%d).standard_normal over the global domain, host-centred "
                       "(sha256 %s...)" % (2 if world == 1 else 3, rhs_sha[:16]),
                # the CPU oracle's iteration count on the same rhs bits (tests/golden/mlmg_golden.json)
                "oracle_iterations": _golden_iterations("c3") if world == 1 else None,
                "oracle_parity": parity,
                "solves": "back to back: step s+1 is queued before step s's result is read "
                          "(MLMG.solve(wait=False) / finish()); each runs its own device-side convergence test",
                "mlmg_solve_ms": ms, "global_batch": 1, "seq_len": dom.num_cells(),
                "parallelism": f"dp{world} (boxes by Morton SFC)",
                "l2": "working set (phi x2 + rhs, 256^3 fp64 per GPU = 0.4 GB) exceeds the 126 MB L2",
            },
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                    "ms_per_step": 1e3 * t_e2e / args.steps,
                    "mode": "pipelined: double-buffered rhs/phi (FabArray host images), step s+1 upload and step s-1 "
                            "download on two copy streams during step s's solve (all copies inside the timed region)",
                    "serial": {"value": e2e_serial, "ms_per_step": 1e3 * t_serial / args.steps},
                    "bounds": {"copies_only_ms_per_step": 1e3 * t_copies / args.steps,
                               "solves_only_ms_per_step": 1e3 * t_solves / args.steps}},
            "roofline": {"bound": "hbm", "kernel": "k_gsrb_stream (fine level, fused red+black, register-streamed, TMA-fed)",
                         "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                         "peak_kind": peak_kind, "traffic": traffic, "alg_bytes_per_launch": alg_bytes,
                         "us_per_launch": t_sweep * 1e6,
                         "kernel_cell_updates_per_s": nloc / t_sweep,
                         # plain fine-level sweeps per solve x this launch time / solve time
                         # (the ncu launch list's share of the same kernel should agree)
                         "launches_per_step": fine_per_step,
                         "share_of_step": fine_per_step * t_sweep / (ms / 1e3)},
            "gpu_launches": int(launches),
            "clocks": clk.summary(),
        }
        if cpu is not None:
            line["cpu_baseline"] = cpu
        if others is not None:
            line["other_configs"] = others
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier(device_ids=[local])


def _graph_us(fn, reps=10):
    """us per call of fn, `reps` calls captured in one CUDA graph (warm)."""
    import torch

    fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        with torch.cuda.graph(g, stream=s):
            for _ in range(reps):
                fn()
    torch.cuda.current_stream().wait_stream(s)
    g.replay()
    torch.cuda.synchronize()
    ts = []
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        g.replay()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3 / reps)
    return float(np.median(ts))


def c1_micro():
    """Config C1: periodic 64^3 in 8 boxes of 32^3, one ghost
    layer; FillBoundary + 7-point Laplacian on the device (graph-timed), and the
    same step in the numpy oracle on the host (the reference's fill_boundary
    measured 2.35 ms)."""
    import torch

    import paper_2009_12009_b200 as A
    from oracle import mesh_ref as M
    from oracle import mlmg_ref as R
    from paper_2009_12009_b200 import stencil as S

    n, m = 64, 32
    dom = A.Box((0, 0, 0), (n - 1,) * 3)
    ba = A.BoxArray([dom]).max_size(m)
    dm = A.DistributionMapping.single_rank(len(ba))
    tr = A.Transport(1)
    g = np.random.default_rng(0).standard_normal((1, n, n, n))
    phi = A.MultiFab(ba, dm, 1, 1)
    phi.setval(-7777.0)
    phi.load_valid_from(dom, g)
    out = A.MultiFab(ba, dm, 1, 0)
    dh = (float(n * n),) * 3
    fill_us = _graph_us(lambda: A.fill_boundary(phi, tr, dom, True))
    lap_us = _graph_us(lambda: S.laplacian(out, phi, dh))
    step_us = _graph_us(lambda: (A.fill_boundary(phi, tr, dom, True), S.laplacian(out, phi, dh)))
    boxes = [(tuple(b.lo), tuple(b.hi)) for b in ba]
    d = ((0, 0, 0), (n - 1,) * 3)
    fabs = M.make_fabs(boxes, 1, 1, -7777.0)
    M.load_global(boxes, fabs, 1, d, g)
    t0 = time.perf_counter()
    reps = 5
    for _ in range(reps):
        M.fill_boundary(boxes, fabs, 1, d, (True,) * 3)
        for i in fabs:
            R.laplacian(fabs[i][0], dh)
    cpu_ms = 1e3 * (time.perf_counter() - t0) / reps
    return {"workload": "C1 periodic 64^3, 8 boxes of 32^3, 1 ghost: FillBoundary + Laplacian",
            "fill_us": round(fill_us, 2), "laplacian_us": round(lap_us, 2), "step_us": round(step_us, 2),
            "cpu_oracle_step_ms": round(cpu_ms, 3), "cpu_oracle": "numpy restatement, 1 thread",
            "timing": "CUDA graph of 10 steps, warm"}


def c5_micro(ghost_push="auto"):
    """Config C5 microtimings (1 GPU): 512^3 in 4,096 boxes of 32^3 -- the
    copy-program FillBoundary at width 1 and 2, the streaming sweep alone and
    with its ghost push, and the bench's C5 step (10 sweeps + Laplacian)."""
    import torch

    import paper_2009_12009_b200 as A
    from paper_2009_12009_b200 import stencil as S
    from paper_2009_12009_b200.ghosts import push_table

    n, m = 512, 32
    dom = A.Box((0, 0, 0), (n - 1,) * 3)
    ba = A.BoxArray([dom]).max_size(m)
    dm = A.DistributionMapping.single_rank(len(ba))
    tr = A.Transport(1)
    a, b = A.MultiFab(ba, dm, 1, 2), A.MultiFab(ba, dm, 1, 2)
    rhs, lap = A.MultiFab(ba, dm, 1, 1), A.MultiFab(ba, dm, 1, 0)
    rng = np.random.default_rng(4)
    a.load_valid_from(dom, rng.standard_normal((n, n, n)))
    rhs.load_valid_from(dom, rng.standard_normal((n, n, n)))
    A.fill_boundary(rhs, tr, dom, True)
    A.fill_boundary(a, tr, dom, True)
    dh = (float(n * n),) * 3
    tab = push_table(b, dom, True, 2)
    tab_a = push_table(a, dom, True, 2)
    res = {"workload": "C5 512^3, 4096 boxes of 32^3, periodic (1 GPU)",
           "fill_w1_us": round(_graph_us(lambda: A.fill_boundary(a, tr, dom, True, ngrow=1)), 1),
           "fill_w2_us": round(_graph_us(lambda: A.fill_boundary(a, tr, dom, True, ngrow=2)), 1),
           "sweep_us": round(_graph_us(lambda: S.gsrb_sweep(a, b, rhs, dh)), 1),
           "sweep_with_ghost_push_us": round(_graph_us(lambda: S.gsrb_sweep(a, b, rhs, dh, push=tab)), 1)}
    fields = [a, b]
    tabs = {id(a): tab_a, id(b): tab}

    def step():
        for _ in range(10):
            S.gsrb_sweep(fields[0], fields[1], rhs, dh, push=tabs[id(fields[1])])
            fields.reverse()
        S.laplacian(lap, fields[0], dh)

    res["step_ms"] = round(_graph_us(step, reps=2) / 1e3, 3)
    res["step"] = "10 x fused sweep (FillBoundary pushed by the sweep) + Laplacian, graph"
    res["cell_updates_per_s"] = 10 * n ** 3 / (res["step_ms"] * 1e-3)
    del a, b, rhs, lap
    torch.cuda.empty_cache()
    return res


def run_c5(args):
    """Config C5: 512^3 in 4,096 boxes of 32^3, periodic; a step =
    10 x (width-2 FillBoundary + fused GSRB sweep) + width-1 FillBoundary +
    Laplacian apply.  N GPUs share the SAME 512^3 problem (strong scaling);
    every rank's boxes by sfc_distribute, fills over NVLink (p2p)."""
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    import paper_2009_12009_b200 as A
    from paper_2009_12009_b200 import stencil as S
    from paper_2009_12009_b200._native import lib
    n, m = 512, 32
    dom = A.Box((0, 0, 0), (n - 1,) * 3)
    ba = A.BoxArray([dom]).max_size(m)
    dm = A.sfc_distribute(ba, A.default_costs(ba), world)
    tr = A.Transport.distributed() if world > 1 else A.Transport(1)
    sym = world > 1
    a = A.MultiFab(ba, dm, 1, 2, symmetric=sym)
    b = A.MultiFab(ba, dm, 1, 2, symmetric=sym)
    rhs = A.MultiFab(ba, dm, 1, 1, symmetric=sym)
    lap = A.MultiFab(ba, dm, 1, 0)
    # phi then rhs, standard normals from np.random.default_rng(4)
    rng = np.random.default_rng(4)
    a.load_valid_from(dom, rng.standard_normal((n, n, n)))
    rhs.load_valid_from(dom, rng.standard_normal((n, n, n)))
    A.fill_boundary(rhs, tr, dom, True)
    dh = (float(n * n),) * 3
    fields = [a, b]
    # FillBoundary fused into the sweep (ghosts.push_table): each sweep also
    # writes its output's width-2 ghosts -- on other GPUs through NVLink, then a
    # device barrier -- instead of a copy-program fill before the next sweep
    # (tools/mb_stream.py, C5 layout: sweep + push 1019 us vs fill + sweep
    # ~1.3 ms); the width-1 fill before the Laplacian is covered as well
    from paper_2009_12009_b200.ghosts import push_table

    tabs = {id(f): push_table(f, dom, True, 2) for f in (a, b)}
    use_push = args.ghost_push != "off" and all(t is not None for t in tabs.values())

    def step():
        for _ in range(10):
            if use_push:
                S.gsrb_sweep(fields[0], fields[1], rhs, dh, push=tabs[id(fields[1])])
                if world > 1:
                    tr.peer_barrier()  # peers' pushes into our ghosts have landed
            else:
                A.fill_boundary(fields[0], tr, dom, True, ngrow=2)
                S.gsrb_sweep(fields[0], fields[1], rhs, dh)
            fields.reverse()
        if not use_push:
            A.fill_boundary(fields[0], tr, dom, True, ngrow=1)
        S.laplacian(lap, fields[0], dh)

    A.fill_boundary(a, tr, dom, True, ngrow=2)  # the first sweep's input

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier(device_ids=[local])
        torch.cuda.synchronize()

    def maxover(x):
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return t.item()

    for _ in range(args.warmup):
        step()
    # capture one step (10 sweeps) in a graph: 4,096-box copy programs are launch-heavy
    barrier()
    g = torch.cuda.CUDAGraph()
    cs = torch.cuda.Stream()
    cs.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(cs):
        with torch.cuda.graph(g, stream=cs, capture_error_mode="relaxed"):
            l0 = lib().amrb_launch_count()
            step()
            per_step = lib().amrb_launch_count() - l0
    torch.cuda.current_stream().wait_stream(cs)
    g.replay()
    barrier()
    st = torch.cuda.current_stream()
    clk = ClockSampler(local)
    clk.__enter__()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for _ in range(args.steps):
        g.replay()
    e1.record(st)
    barrier()
    clk.__exit__(None, None, None)
    t = maxover(e0.elapsed_time(e1) / 1e3)
    ncells = dom.num_cells()
    value = 10 * ncells * args.steps / t
    # e2e: phi in from pinned host memory (data.bin image: one copy + one
    # scatter launch), the step, phi back out (one gather launch + one copy)
    nbytes = 8 * a.image_size()
    host_in = torch.empty(a.image_size(), dtype=torch.float64).pin_memory()
    host_out = torch.empty(a.image_size(), dtype=torch.float64).pin_memory()
    a.to_host_image(host_in)
    a.from_host_image(host_in)  # untimed: builds the image staging + programs
    barrier()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        a.from_host_image(host_in)
        if use_push:  # the uploaded phi's ghosts (the graph's sweeps keep them current after this)
            A.fill_boundary(a, tr, dom, True, ngrow=2)
        fields[:] = [a, b]
        g.replay()
        a.to_host_image(host_out)
        torch.cuda.synchronize()
    barrier()
    t_e2e = maxover(time.perf_counter() - t0)
    # roofline: the sweep alone on this layout (N valid cells, F face ghosts of 32^3 boxes)
    evs = []
    for _ in range(8):
        A.fill_boundary(a, tr, dom, True, ngrow=2)
        s0 = torch.cuda.Event(enable_timing=True)
        s1 = torch.cuda.Event(enable_timing=True)
        s0.record(st)
        S.gsrb_sweep(a, b, rhs, dh)
        s1.record(st)
        evs.append((s0, s1))
    torch.cuda.synchronize()
    t_sw = maxover(float(np.mean([x.elapsed_time(y) for x, y in evs[3:]])) / 1e3)
    nloc = sum(ba[i].num_cells() for i in range(len(ba)) if dm[i] == rank)
    floc = sum(6 * m * m for i in range(len(ba)) if dm[i] == rank)
    alg = 24 * nloc + 8 * floc
    peak, peak_kind = _peaks()
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = _c5_cpu_sample()
    if rank == 0:
        line = {
            "metric": "fp64 cell-updates/s (C5: 10 GSRB sweeps + Laplacian, 512^3 in 32^3 boxes)", "value": value,
            "unit": UNIT, "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * t / args.steps, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic",
            "config": {"workload": "C5 512^3, 4096 boxes of 32^3, periodic: 10 x (fill w2 + fused GSRB sweep) + "
                                   "fill w1 + Laplacian per step (one CUDA graph)", "domain": [n] * 3, "box": m,
                       "fill": ("fused into the sweep (ghost push" + (", NVLink + device barrier" if world > 1 else "")
                                + ")") if use_push else "copy-program FillBoundary",
                       "boxes": len(ba), "global_batch": 1, "seq_len": ncells,
                       "parallelism": f"dp{world} (boxes by Morton SFC, same problem on every GPU count)",
                       "l2": "working set 5+ GB exceeds the 126 MB L2"},
            "e2e": {"value": 10 * ncells * args.steps / t_e2e, "unit": UNIT, "h2d_bytes_per_step": nbytes,
                    "d2h_bytes_per_step": nbytes, "ms_per_step": 1e3 * t_e2e / args.steps,
                    "mode": "serial: phi image in (FabArray.from_host_image), step, phi image out"},
            "roofline": {"bound": "hbm", "kernel": "GSRB sweep on 32^3 boxes", "achieved": alg / t_sw / 1e9,
                         "peak": peak, "unit": "GB/s", "frac": alg / t_sw / 1e9 / peak, "peak_kind": peak_kind,
                         "traffic": None, "alg_bytes_per_launch": alg, "us_per_launch": t_sw * 1e6},
            "gpu_launches": int(per_step) * args.steps,
            "clocks": clk.summary(),
        }
        if cpu is not None:
            line["cpu_baseline"] = cpu
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier(device_ids=[local])


def _c5_cpu_sample():
    """Oracle GSRB sweeps (fill, red, fill, black) on a 256^3 domain of C5's
    32^3 boxes, colour updates on every host thread (a few seconds)."""
    from oracle import mesh_ref as M
    from oracle import mlmg_ref as R

    n, m = 256, 32
    boxes = [((i, j, k), (i + m - 1, j + m - 1, k + m - 1)) for i in range(0, n, m) for j in range(0, n, m)
             for k in range(0, n, m)]
    dom = ((0, 0, 0), (n - 1,) * 3)
    phi = M.make_fabs(boxes, 1, 1)
    rhs = M.make_fabs(boxes, 1, 0)
    rng = np.random.default_rng(4)
    for f in list(phi.values()) + list(rhs.values()):
        f[...] = rng.standard_normal(f.shape)
    recs = M.fill_records(boxes, 1, dom, (True, True, True))
    dh = (512.0 * 512.0,) * 3
    from concurrent.futures import ThreadPoolExecutor

    threads = os.cpu_count() or 1
    t0 = time.perf_counter()
    sweeps = 2
    with ThreadPoolExecutor(threads) as pool:
        for _ in range(sweeps):
            for color in (0, 1):
                M.execute(recs, boxes, phi, 1, boxes, phi, 1)
                list(pool.map(lambda i: R.gsrb_color(boxes[i], phi[i][0], rhs[i][0], dh, color), range(len(boxes))))
    dt = time.perf_counter() - t0
    return {"value": sweeps * n ** 3 / dt, "unit": UNIT, "cores": threads, "kind": "port",
            "sample": f"{sweeps} oracle GSRB sweeps (fill, red, fill, black) over 256^3 in 512 boxes of 32^3 "
                      f"({dt:.1f} s; per-box colour updates on {threads} threads, fills serial)"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-other-configs", action="store_true", help="skip the C1 / C5 microtimings of the C3 line")
    ap.add_argument("--ghost-push", default="auto", choices=["auto", "on", "off", "remote"],
                    help="A/B runs: MLMG ghost push (auto: across GPUs only)")
    ap.add_argument("--option", action="append", default=[], metavar="NAME=VALUE",
                    help="A/B runs: set a library option (amrb_set_option) before building")
    ap.add_argument("--config", default="c3", choices=["c3", "c5"],
                    help="c3: the headline MLMG solve (C3 / C4 weak scaling); c5: 512^3 sweeps (strong scaling)")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.option:
        from paper_2009_12009_b200._native import set_option

        for kv in args.option:
            name, _, value = kv.partition("=")
            set_option(name, int(value))
    if args.impl == "reference":
        run_reference(args)
    elif args.config == "c5":
        run_c5(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
