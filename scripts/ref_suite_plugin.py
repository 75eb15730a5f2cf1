"""pytest plugin: run the REFERENCE's own test suite (baseline/_ref/tests,
the unmodified reference package installed into baseline/_ref) with the
B200 proximity path installed through ``rfx_compat.install`` — every call
the suite makes to rfx.proximity.{leaf_membership, full_proximity,
triblock_proximity, lowrank_proximity, outlier_scores} and
rfx.mds.{gram_matvec, mds_lowrank} runs on the GPU.

    python -m pytest -p ref_suite_plugin baseline/_ref/tests   (scripts/ on sys.path)

At the end it prints how many calls each patched function served and how
many librfxc kernels were launched, so a pass cannot come from the CPU path.
"""

import collections
import functools
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for p in (os.path.join(ROOT, "baseline", "_ref"), ROOT):
    if p not in sys.path:
        sys.path.insert(0, p)

import rfx  # noqa: E402
import rfx.mds  # noqa: E402
import rfx.proximity  # noqa: E402

from paper_2511_19493_b200 import _lib, rfx_compat  # noqa: E402

rfx_compat.install(rfx)
CALLS = collections.Counter()
for modname, names in rfx_compat.PATCHED.items():
    mod = getattr(rfx, modname)
    for name in names:
        fn = getattr(mod, name)

        def counted(*a, _fn=fn, _key=f"{modname}.{name}", **kw):
            CALLS[_key] += 1
            return _fn(*a, **kw)
        setattr(mod, name, functools.wraps(fn)(counted))


def pytest_terminal_summary(terminalreporter):
    tr = terminalreporter
    tr.write_sep("=", "B200 path served (rfx_compat.install)")
    for key in sorted(CALLS):
        tr.write_line(f"  {key:36s} {CALLS[key]:6d} calls")
    tr.write_line(f"  librfxc kernel launches: {_lib.launch_count}")
    tr.write_line(f"  library: {_lib.LIB_PATH}")
