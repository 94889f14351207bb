"""ctypes binding of libamrb.so (include/amrb.h).

The library is built in-tree by ``__graft_entry__.build()`` (or ``make -C
paper_2009_12009_b200/csrc``).  There is no fallback: if the shared object is
missing, every device operation raises.
"""

from __future__ import annotations

import ctypes as C
import os
import threading

import numpy as np

__all__ = ["lib", "check", "LIB_PATH", "AmrbError", "ptr", "i32p", "i64p", "u8p", "f64p", "get_option", "set_option",
           "option"]

# AMRB_LIBRARY=checked selects the checked build (device invariant checks,
# make -C csrc CHECKED=1) for test runs; the default is the production library
LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "_lib",
                        "libamrb_checked.so" if os.environ.get("AMRB_LIBRARY") == "checked" else "libamrb.so")

AMRB_OK, AMRB_EINVAL, AMRB_ECUDA, AMRB_ENCCL, AMRB_ENOMEM, AMRB_ENOTSUP = 0, -1, -2, -3, -4, -5
FABTAB_W = 8
REC_W = 11


class AmrbError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(msg)
        self.code = code


vp = C.c_void_p
i32, i64, f64 = C.c_int32, C.c_int64, C.c_double
P = C.POINTER

_SIGS = {
    "amrb_last_error": (C.c_char_p, []),
    "amrb_version": (C.c_int, []),
    "amrb_launch_count": (i64, []),
    "amrb_loop_begin": (C.c_int, [vp, P(vp)]),
    "amrb_loop_reset": (C.c_int, [vp, C.c_double, C.c_int, vp, vp]),
    "amrb_loop_control": (C.c_int, [vp, vp, vp, vp, C.c_int, vp]),
    "amrb_loop_end": (C.c_int, [vp]),
    "amrb_loop_launch": (C.c_int, [vp, vp]),
    "amrb_loop_destroy": (C.c_int, [vp]),
    "amrb_debug_checks": (C.c_int, [P(i64), P(i64), C.c_int]),
    "amrb_set_option": (C.c_int, [C.c_char_p, i64]),
    "amrb_get_option": (C.c_int, [C.c_char_p, P(i64)]),
    "amrb_zero": (C.c_int, [vp, i64, vp]),
    "amrb_fill": (C.c_int, [vp, i64, f64, vp]),
    "amrb_fill_wrap": (C.c_int, [vp, vp, vp, C.c_int, C.c_int, vp]),
    "amrb_setval": (C.c_int, [vp, vp, vp, C.c_int, C.c_int, C.c_int, C.c_int, f64, vp]),
    "amrb_store_host": (C.c_int, [vp, vp, i64, vp]),
    "amrb_morton_key": (C.c_int, [C.c_int, P(i32), P(i32), P(C.c_uint64)]),
    "amrb_sfc_distribute": (C.c_int, [C.c_int, C.c_int, P(i32), P(f64), f64, C.c_int, P(i32)]),
    "amrb_knapsack_distribute": (C.c_int, [C.c_int, P(f64), C.c_int, P(i32)]),
    "amrb_plan_fill_create": (C.c_int, [C.c_int, C.c_int, P(i32), C.c_int, P(i32), P(C.c_uint8), P(vp)]),
    "amrb_plan_copy_create": (
        C.c_int,
        [C.c_int, C.c_int, P(i32), C.c_int, P(i32), C.c_int, P(i32), P(C.c_uint8), P(vp)],
    ),
    "amrb_plan_sum_create": (C.c_int, [C.c_int, C.c_int, P(i32), C.c_int, P(i32), P(C.c_uint8), P(vp)]),
    "amrb_plan_size": (C.c_int, [vp, P(i64), P(i64)]),
    "amrb_plan_records": (C.c_int, [vp, P(i32)]),
    "amrb_plan_destroy": (C.c_int, [vp]),
    "amrb_prog_create": (
        C.c_int,
        [vp, C.c_int, P(i64), C.c_int, P(i32), P(i64), C.c_int, P(i32), C.c_int, C.c_int, C.c_int, C.c_int, P(vp)],
    ),
    "amrb_prog_info": (C.c_int, [vp, P(i64), P(i64), P(i64), P(i64)]),
    "amrb_prog_pairs": (C.c_int, [vp, P(i64)]),
    "amrb_prog_run": (C.c_int, [vp, vp, vp, vp, vp, vp, vp]),
    "amrb_prog_destroy": (C.c_int, [vp]),
    "amrb_prog_run_p2p": (C.c_int, [vp, vp, vp, P(C.c_uint64), C.c_int, vp]),
    "amrb_prog_run_p2p_sync": (C.c_int, [vp, vp, vp, P(C.c_uint64), C.c_int, P(C.c_uint64), C.c_int, vp, vp]),
    "amrb_set_fault_mailbox": (C.c_int, [vp]),
    "amrb_peer_barrier": (C.c_int, [P(C.c_uint64), C.c_int, C.c_int, vp, vp]),
    "amrb_peer_allmax": (C.c_int, [P(C.c_uint64), P(C.c_uint64), C.c_int, C.c_int, vp, vp, vp]),
    "amrb_level_create": (C.c_int, [C.c_int, P(i32), P(C.c_uint8), P(vp)]),
    "amrb_level_destroy": (C.c_int, [vp]),
    "amrb_field_create": (C.c_int, [vp, P(i64), C.c_int, P(vp)]),
    "amrb_field_destroy": (C.c_int, [vp]),
    "amrb_lap_apply": (C.c_int, [vp, vp, vp, vp, vp, P(f64), vp]),
    "amrb_residual": (C.c_int, [vp, vp, vp, vp, vp, vp, vp, P(f64), vp]),
    "amrb_gsrb_color": (C.c_int, [vp, vp, vp, vp, vp, P(f64), C.c_int, vp]),
    "amrb_gsrb_sweep": (C.c_int, [vp, vp, vp, vp, vp, vp, vp, P(f64), P(i32), vp, vp]),
    "amrb_gsrb_sweep_norm": (C.c_int, [vp, vp, vp, vp, vp, vp, vp, P(f64), P(i32), vp, vp, vp]),
    "amrb_gsrb_sweep_pull": (C.c_int, [vp, vp, vp, vp, vp, vp, vp, P(f64), vp, vp, C.c_int, C.c_int, vp, vp, vp]),
    "amrb_gsrb_sweep_prolong": (C.c_int, [vp, vp, vp, vp, vp, vp, vp, P(f64), vp, vp, vp, vp, vp]),
    "amrb_restrict": (C.c_int, [vp, vp, vp, vp, vp, C.c_int, P(i32), C.c_int, vp]),
    "amrb_residual_restrict": (C.c_int, [vp, vp, vp, vp, vp, vp, vp, P(f64), vp]),
    "amrb_prolong": (C.c_int, [vp, vp, vp, vp, vp, C.c_int, P(i32), C.c_int, vp]),
    "amrb_adv_flux": (C.c_int, [vp, vp, vp, vp, vp, C.c_int, i64, vp, vp, C.c_int, C.c_int, f64, vp]),
    "amrb_adv_update": (C.c_int, [vp, vp, vp, vp, vp, C.c_int, i64, vp, vp, C.c_int, C.c_int, P(f64), vp]),
    "amrb_axpby": (C.c_int, [vp, vp, vp, C.c_int, i64, vp, vp, f64, vp, vp, f64, vp, vp, vp]),
    "amrb_interp": (C.c_int, [vp, vp, vp, vp, vp, vp, vp, vp, C.c_int, i64, C.c_int, C.c_int, P(i32), C.c_int, vp]),
    "amrb_nan_count": (C.c_int, [vp, vp, vp, vp, C.c_int, i64, vp, C.c_int, vp, vp]),
    "amrb_fr_crse": (C.c_int, [vp, i64, vp, vp, f64, vp]),
    "amrb_fr_fine": (C.c_int, [vp, i64, C.c_int, C.c_int, vp, vp, f64, vp]),
    "amrb_fr_reflux": (C.c_int, [vp, vp, i64, vp, vp, vp, vp, vp]),
    "amrb_reduce": (C.c_int, [vp, vp, vp, C.c_int, C.c_int, vp, vp]),
    "amrb_residual_norm": (C.c_int, [vp, vp, vp, vp, vp, P(f64), vp, vp]),
    "amrb_coarse_tail": (C.c_int, [C.c_int, P(i32), P(f64), vp, vp, vp, vp, C.c_int, C.c_int, C.c_int, C.c_int,
                                   P(i32), vp]),
    "amrb_level_grid": (C.c_int, [C.c_int, P(i32), P(f64), vp, vp, vp, vp, vp, vp, C.c_int, vp]),
    "amrb_domain_bc": (C.c_int, [vp, vp, vp, C.c_int, P(i32), P(i32), f64, vp]),
    "amrb_nccl_unique_id": (C.c_int, [P(C.c_uint8)]),
    "amrb_nccl_comm_create": (C.c_int, [P(C.c_uint8), C.c_int, C.c_int, P(vp)]),
    "amrb_nccl_comm_destroy": (C.c_int, [vp]),
    "amrb_nccl_allreduce": (C.c_int, [vp, i64, C.c_int, vp, vp]),
    "amrb_nccl_allgather": (C.c_int, [vp, vp, i64, vp, vp]),
}

EXPORTED = tuple(_SIGS)

_lib = None
_lock = threading.Lock()


def lib():
    """The loaded library; raises if it was never built (no CPU fallback)."""
    global _lib
    if _lib is None:
        with _lock:
            if _lib is None:
                if not os.path.exists(LIB_PATH):
                    raise RuntimeError(
                        f"libamrb.so not built ({LIB_PATH}); run __graft_entry__.build() "
                        "or `make -C paper_2009_12009_b200/csrc` -- there is no CPU fallback"
                    )
                handle = C.CDLL(LIB_PATH)
                for name, (res, args) in _SIGS.items():
                    fn = getattr(handle, name)
                    fn.restype = res
                    fn.argtypes = args
                _lib = handle
    return _lib


def check(status, *, src=None, dst=None):
    """Map a status code to the reference's exception types."""
    if status == AMRB_OK:
        return
    msg = lib().amrb_last_error().decode(errors="replace")
    if status == AMRB_EINVAL:
        raise ValueError(msg)
    if status == AMRB_ENCCL:
        from .comm import TransportError

        raise TransportError(src if src is not None else -1, dst if dst is not None else -1, msg)
    raise AmrbError(status, msg)


def ptr(x):
    """Raw address of a torch tensor / numpy array (None -> NULL)."""
    if x is None:
        return None
    if hasattr(x, "data_ptr"):
        return x.data_ptr()
    return x.ctypes.data


def _np_ptr(a, ctype):
    return a.ctypes.data_as(P(ctype))


def i32p(a):
    a = np.ascontiguousarray(a, dtype=np.int32)
    return a, _np_ptr(a, i32)


def i64p(a):
    a = np.ascontiguousarray(a, dtype=np.int64)
    return a, _np_ptr(a, i64)


def u8p(a):
    a = np.ascontiguousarray(a, dtype=np.uint8)
    return a, _np_ptr(a, C.c_uint8)


def f64p(a):
    a = np.ascontiguousarray(a, dtype=np.float64)
    return a, _np_ptr(a, f64)


def get_option(name):
    """Current value of a library option (include/amrb.h amrb_set_option)."""
    v = i64(0)
    check(lib().amrb_get_option(name.encode(), C.byref(v)))
    return int(v.value)


def set_option(name, value):
    """Set a library option; returns the previous value."""
    old = get_option(name)
    check(lib().amrb_set_option(name.encode(), int(value)))
    return old


class option:
    """``with option("sweep_kernel", 1): ...`` -- scoped library option (A/B runs, tests)."""

    def __init__(self, name, value):
        self.name, self.value = name, value

    def __enter__(self):
        self.old = set_option(self.name, self.value)
        return self

    def __exit__(self, *exc):
        set_option(self.name, self.old)


def debug_checks(reset=True):
    """(failures, first failing source line) of the checked build's device
    invariant checks; failures = -1 in the production build."""
    f, ln = i64(0), i64(0)
    check(lib().amrb_debug_checks(C.byref(f), C.byref(ln), 1 if reset else 0))
    return int(f.value), int(ln.value)
