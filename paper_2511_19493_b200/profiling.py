"""Per-kernel CUDA-event timing on the launching stream (bench.py uses it to
measure the dominant kernel's average launch duration inside the timed
region).  Disabled by default: the hooks cost nothing when off."""

from __future__ import annotations

import contextlib
from collections import defaultdict

_active = None


class KernelTimer:
    def __init__(self):
        self.events = defaultdict(list)
        self.launches = defaultdict(int)

    def elapsed_ms(self):
        """{name: (total_ms, launches)} — call after synchronising."""
        out = {}
        for name, pairs in self.events.items():
            out[name] = (sum(a.elapsed_time(b) for a, b in pairs), len(pairs))
        return out


def start():
    global _active
    _active = KernelTimer()
    return _active


def stop():
    global _active
    t, _active = _active, None
    return t


@contextlib.contextmanager
def region(name: str):
    """Bracket one launch (or a group of launches) with CUDA events."""
    if _active is None:
        yield
        return
    import torch
    a = torch.cuda.Event(enable_timing=True)
    b = torch.cuda.Event(enable_timing=True)
    a.record()
    try:
        yield
    finally:
        b.record()
        _active.events[name].append((a, b))
