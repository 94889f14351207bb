"""Golden MLMG solves at the headline configs (C2, C3) from the CPU oracle.

TEST INFRASTRUCTURE.  Run in the build container (numpy only, ~1 min on 8
threads):

    python tests/golden/make_mlmg_golden.py

For each config it builds the synthetic rhs exactly as SURVEY.md 8(d) and
bench.py do (``np.random.default_rng(seed).standard_normal`` over the global
domain, host-centred), solves it with ``oracle.mlmg_ref.OracleMLMG`` on the
box layout of the config, and stores in ``mlmg_golden.json``:

* ``rhs_sha256``  -- sha256 of the centred rhs (C-order float64 bytes), so a
  GPU test can prove it solves the same bits;
* ``iterations``, ``history`` (float.hex, exact), ``r0``;
* ``phi_sha256``  -- sha256 of the converged solution (gathered global array);
* ``phi_probe``   -- phi on a coarse lattice (every 16th cell, float.hex) to
  localise a mismatch without shipping the 134 MB solution.

The GPU test (tests/test_gpu_mlmg_headline.py) solves the same rhs through
``MLMG.solve`` and compares all of these bit for bit.
"""

from __future__ import annotations

import hashlib
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))

# (name, domain extent, box size, seed, bc) -- SURVEY.md 8(d) C2 / C3, plus the
# Dirichlet (external, value 0) variant of C2 (amr_core.py:73-146)
CASES = [
    ("c2", 128, 32, 1, "periodic"),
    ("c3", 256, 64, 2, "periodic"),
    ("c2_dirichlet", 128, 32, 1, "dirichlet"),
]
PROBE = 16


def headline_rhs(n, seed, centre=True):
    """The synthetic rhs of SURVEY 8(d): seeded standard normals on the global
    n^3 array (or an (n0, n1, n2) shape), minus their host mean (periodic: the
    singular problem needs a zero-mean rhs; every arm sees identical bits)."""
    shape = (n, n, n) if np.isscalar(n) else tuple(n)
    rhs = np.random.default_rng(seed).standard_normal(shape)
    if centre:
        rhs -= rhs.mean()
    return rhs


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.float64).tobytes()).hexdigest()


def probe(phi):
    return [float(x).hex() for x in phi[::PROBE, ::PROBE, ::PROBE].ravel()]


def boxes_of(n, m):
    return [((i, j, k), (i + m - 1, j + m - 1, k + m - 1)) for i in range(0, n, m) for j in range(0, n, m)
            for k in range(0, n, m)]


def main():
    sys.path.insert(0, ROOT)
    from oracle import mlmg_ref as R

    out = {}
    threads = os.cpu_count() or 1
    for name, n, m, seed, bc in CASES:
        rhs = headline_rhs(n, seed, centre=bc == "periodic")
        t0 = time.perf_counter()
        s = R.OracleMLMG(((0, 0, 0), (n - 1,) * 3), boxes_of(n, m), threads=threads, bc=bc)
        res = s.solve(rhs, rtol=1e-10, max_iter=200)
        dt = time.perf_counter() - t0
        out[name] = {
            "n": n, "box": m, "seed": seed, "bc": bc, "rtol": 1e-10,
            "rhs_sha256": sha(rhs),
            "iterations": res["iterations"],
            "history": [float(x).hex() for x in res["history"]],
            "r0": float(res["r0"]).hex(),
            "phi_sha256": sha(res["phi"]),
            "phi_probe_stride": PROBE,
            "phi_probe": probe(res["phi"]),
        }
        print(f"{name}: {res['iterations']} cycles, final {res['history'][-1]:.3e} (r0 {res['r0']:.3e}), "
              f"{dt:.1f} s on {threads} threads", flush=True)
    with open(os.path.join(HERE, "mlmg_golden.json"), "w") as f:
        json.dump(out, f, indent=1)
        f.write("\n")


if __name__ == "__main__":
    main()
