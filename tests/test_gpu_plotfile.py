"""Device plotfile / checkpoint writer: byte-identical to the
reference's write_plotfile (golden digests made by tests/golden/make_golden.py
from amrkit itself), independent of rank count, writer count and sync/async
mode; bitwise round trip; async snapshot isolation."""

import json
import os
import sys
import types

import numpy as np
import pytest
import torch

import paper_2009_12009_b200 as A

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden"))
import plotfile_cases as PC  # noqa: E402

pytestmark = pytest.mark.gpu

GOLD = json.load(open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "plotfile.json")))
NS = types.SimpleNamespace(Box=A.Box, IntVect=A.IntVect, BoxArray=A.BoxArray, Geometry=A.Geometry,
                           FabArray=A.FabArray, sfc_distribute=A.sfc_distribute, default_costs=A.default_costs,
                           PlotfileHeader=A.PlotfileHeader)


@pytest.mark.parametrize("case", PC.CASES, ids=[c[0] for c in PC.CASES])
def test_bytes_match_reference(case, tmp_path):
    header, meshes = PC.build(NS, case)
    for kind, mode in (("s1", A.OutputMode.static(1)), ("s3", A.OutputMode.static(3)),
                       ("async", A.OutputMode.asynchronous())):
        path = str(tmp_path / f"plt_{kind}")
        A.write_plotfile(path, meshes, header, mode).wait()
        with open(os.path.join(path, "Header")) as fh:
            assert fh.read() == GOLD[case[0]]["header"]
        assert PC.dir_digest(path) == GOLD[case[0]]["digest"], kind


def test_round_trip_bitwise(tmp_path):
    case = PC.CASES[1]
    header, meshes = PC.build(NS, case)
    path = str(tmp_path / "plt")
    A.write_plotfile(path, meshes, header).wait()
    got_h, got_m = A.read_plotfile(path)
    assert got_h.time == header.time and got_h.names == header.names
    for lev in range(len(meshes)):
        dom = header.geoms[lev].domain
        assert got_h.geoms[lev].domain == dom
        for c in range(len(header.names)):
            assert np.array_equal(A.gather_global(got_m[lev], dom, comp=c), A.gather_global(meshes[lev], dom, comp=c))


def test_async_snapshot_isolation(tmp_path):
    header, meshes = PC.build(NS, PC.CASES[0])
    want = [A.gather_global(m, g.domain) for m, g in zip(meshes, header.geoms)]
    path = str(tmp_path / "plt")
    h = A.write_plotfile(path, meshes, header, A.OutputMode.asynchronous())
    for m in meshes:  # overwrite on the device right after submit
        m.storage.fill_(-1234.5)
    h.wait()
    assert h.done
    _, got = A.read_plotfile(path)
    for lev in range(len(meshes)):
        assert np.array_equal(A.gather_global(got[lev], header.geoms[lev].domain), want[lev])


def test_wave_counters(tmp_path):
    header, meshes = PC.build(NS, PC.CASES[1])  # 4 simulated ranks
    A.counters.reset("io_waves", "io_peak_writers", "io_bytes_written")
    A.write_plotfile(str(tmp_path / "p2"), meshes, header, A.OutputMode.static(2)).wait()
    assert A.counters.get("io_waves") == 2 * len(meshes)
    assert A.counters.get("io_peak_writers") == 2
    assert A.counters.get("io_bytes_written") == sum(8 * m.ncomp * m.ba.num_cells() for m in meshes)
    A.counters.reset("io_waves", "io_peak_writers")
    A.write_plotfile(str(tmp_path / "p1"), meshes, header, A.OutputMode.static(1)).wait()
    assert A.counters.get("io_waves") == 4 * len(meshes) and A.counters.get("io_peak_writers") == 1


def test_checkpoint_round_trip(tmp_path):
    header, meshes = PC.build(NS, PC.CASES[2])
    blob = b"\x00solver state\xff"
    c1 = str(tmp_path / "c1")
    A.write_checkpoint(c1, meshes, header, step=9, user_blob=blob)
    data = A.read_checkpoint(c1)
    assert data["step"] == 9 and data["blob"] == blob and data["time"] == header.time
    assert data["owners"] == [list(meshes[0].dm.owner)]
    dom = header.geoms[0].domain
    assert np.array_equal(A.gather_global(data["meshes"][0], dom), A.gather_global(meshes[0], dom))
    assert PC.dir_digest(os.path.join(c1, "mesh")) == GOLD[PC.CASES[2][0]]["digest"]
    with pytest.raises(ValueError):
        A.write_checkpoint(str(tmp_path / "c2"), meshes, header, step=1, pc=object())
