"""Shared fixtures.  GPU tests carry @pytest.mark.gpu; the rest run on CPU."""

import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
HERE = os.path.dirname(os.path.abspath(__file__))
if HERE not in sys.path:
    sys.path.insert(0, HERE)

REFERENCE_SRC = "/root/reference/pkg/src"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")


def pytest_collection_modifyitems(config, items):
    import torch

    if torch.cuda.is_available():
        return
    skip = pytest.mark.skip(reason="no CUDA device")
    for it in items:
        if "gpu" in it.keywords:
            it.add_marker(skip)


@pytest.fixture
def rng():
    return np.random.default_rng(20260819)


@pytest.fixture(scope="session")
def amrkit():
    """The unmodified reference package (only in the build container)."""
    if not os.path.isdir(REFERENCE_SRC):
        pytest.skip("reference sources not present (GPU box)")
    if REFERENCE_SRC not in sys.path:
        sys.path.append(REFERENCE_SRC)
    import amrkit as ak

    return ak


def pytest_sessionfinish(session, exitstatus):
    """Under the checked build (AMRB_LIBRARY=checked) report the device-side
    invariant checks the whole session recorded (csrc/device.h AMRB_DCHECK)."""
    if os.environ.get("AMRB_LIBRARY") != "checked":
        return
    try:
        import torch

        if not torch.cuda.is_available():
            return
        from paper_2009_12009_b200._native import debug_checks

        fails, line = debug_checks(reset=False)
        print(f"\nlibamrb_checked.so: session DCHECK failures {fails} (first at line {line})")
        if fails:
            session.exitstatus = 1
    except Exception as e:  # report, do not mask the test outcome
        print(f"\nchecked-build report unavailable: {e}")
