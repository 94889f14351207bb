"""Test helpers: seeded layouts and conversions between the package's Box
types and the oracle's tuple boxes."""

import numpy as np

import paper_2009_12009_b200 as A


def random_cover(rng, domain, nsplits=6):
    """Disjoint BoxArray covering ``domain`` by repeated random axis cuts."""
    pieces = [domain]
    for _ in range(nsplits):
        k = int(rng.integers(len(pieces)))
        b = pieces[k]
        e = b.extents()
        axes = [d for d in range(b.dim) if e[d] >= 2]
        if not axes:
            continue
        d = axes[int(rng.integers(len(axes)))]
        cut = b.lo[d] + int(rng.integers(1, e[d]))
        hi_a = list(b.hi)
        hi_a[d] = cut - 1
        lo_b = list(b.lo)
        lo_b[d] = cut
        pieces[k : k + 1] = [A.Box(b.lo, hi_a), A.Box(lo_b, b.hi)]
    return A.BoxArray(pieces)


def cube(n, dim=3, lo=0):
    return A.Box([lo] * dim, [lo + n - 1] * dim)


def tbox(b):
    return (tuple(b.lo), tuple(b.hi))


def tboxes(ba):
    return [tbox(b) for b in ba]


def wrap(idx, domain, periodic):
    """Source cell of a ghost cell under the domain's wrap, or None."""
    out = []
    for d in range(domain.dim):
        e = domain.extents()[d]
        c = idx[d] - domain.lo[d]
        if periodic[d]:
            out.append(c % e)
        elif 0 <= c < e:
            out.append(c)
        else:
            return None
    return tuple(out)


def oracle_fabs_from_device(fa):
    """{i: numpy array of the fab's full (ncomp, grown) data}."""
    return {i: f.data.cpu().numpy().copy() for i, f in fa.fabs.items()}


def load_device_from_oracle(fa, fabs):
    import torch

    for i, f in fa.fabs.items():
        f.data.copy_(torch.as_tensor(fabs[i]))
