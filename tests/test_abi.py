"""The C-ABI library loads without a GPU and exports every symbol that
include/rfxc.h declares; the ctypes table matches the header."""

import ctypes
import os
import re

from conftest import ROOT


def header_functions():
    text = open(os.path.join(ROOT, "include", "rfxc.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(rfxc_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_entry_points():
    names = header_functions()
    for must in ("rfxc_leaf_codes", "rfxc_bucket", "rfxc_pair_counts", "rfxc_leaf_sums",
                 "rfxc_leaf_gather", "rfxc_factor_quantize", "rfxc_pmax", "rfxc_mds_power"):
        assert must in names


def test_library_exports_every_declared_symbol(built):
    from paper_2511_19493_b200 import _lib
    lib = ctypes.CDLL(_lib.LIB_PATH)
    missing = [n for n in header_functions() if not hasattr(lib, n)]
    assert not missing, missing


def test_ctypes_table_matches_header(built):
    from paper_2511_19493_b200 import _lib
    assert sorted(_lib.SIGNATURES) == header_functions()
    _lib.load()  # binds every argtype without creating a CUDA context
    assert _lib.load().rfxc_version() == 1


def test_argument_counts_match_header(built):
    from paper_2511_19493_b200 import _lib
    text = open(os.path.join(ROOT, "include", "rfxc.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    for name, (_res, args) in _lib.SIGNATURES.items():
        m = re.search(name + r"\s*\(([^)]*)\)", text)
        params = [p for p in m.group(1).split(",") if p.strip() and p.strip() != "void"]
        assert len(params) == len(args), name


def test_sm100a_cubin_present(built):
    """The library carries sm_100a SASS (not just PTX)."""
    import subprocess
    from paper_2511_19493_b200 import _lib
    out = subprocess.run(["cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def test_error_mapping(built):
    import pytest
    from paper_2511_19493_b200 import _lib
    from paper_2511_19493_b200.errors import BudgetError, DataError, RfxError
    with pytest.raises(DataError):
        _lib.check(_lib.RFXC_EDATA, "x")
    with pytest.raises(BudgetError):
        _lib.check(_lib.RFXC_EBUDGET, "x")
    with pytest.raises(RfxError):
        _lib.check(_lib.RFXC_ECUDA, "x")
    # a shape error is reported before any device work
    rc = _lib.load().rfxc_pair_counts(None, 1, 1, 0, 1, 0, None, None, None)
    assert rc == _lib.RFXC_EDATA and b"bad shape" in _lib.load().rfxc_last_error()
