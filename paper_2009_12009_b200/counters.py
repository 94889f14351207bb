"""Named integer tallies shared by the whole process.

Same names and meaning as the reference's instrumentation
(/root/reference/pkg/src/amrkit/counters.py:18-47): ``plans_built``,
``transport_messages``, ``transport_bytes``, ``hash_bins_examined`` and
``hash_queries`` are asserted on by the ghost-exchange tests, so traffic is
checked by counting rather than timing.
"""

from __future__ import annotations

import threading
from collections import Counter

__all__ = ["incr", "peak", "get", "snapshot", "reset"]

_guard = threading.Lock()
_tally: Counter = Counter()


def incr(name, amount=1):
    with _guard:
        _tally[name] += amount


def peak(name, value):
    """Keep the running maximum under ``name``."""
    with _guard:
        _tally[name] = max(_tally[name], value)


def get(name):
    with _guard:
        return _tally[name]


def snapshot():
    with _guard:
        return dict(_tally)


def reset(*names):
    """Zero the given tallies, or all of them when called without names."""
    with _guard:
        if not names:
            _tally.clear()
        for n in names:
            _tally[n] = 0
