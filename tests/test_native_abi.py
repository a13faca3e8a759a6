"""The C-ABI library loads and exports every entry point include/pt_b200.h declares.

CPU-only: no compute calls (the container has no GPU); error paths that fail
before touching a device are exercised.
"""

import ctypes as C
import re
from pathlib import Path

import pytest

from paper_1410_5910_b200 import _native as nat

HEADER = Path(__file__).resolve().parents[1] / "include" / "pt_b200.h"


def declared():
    text = HEADER.read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(pt_[A-Za-z_0-9]+)\s*\(", text)))


def test_header_declares_the_boundary():
    names = declared()
    for must in ("pt_create", "pt_destroy", "pt_apply_A", "pt_apply_M", "pt_gs_sweep",
                 "pt_gmres", "pt_gmres_host", "pt_gmres_batch", "pt_last_error"):
        assert must in names


def test_library_exports_every_declared_symbol():
    lib = nat.lib()
    missing = [n for n in declared() if not hasattr(lib, n)]
    assert not missing, missing
    # and the Python binding covers all of them
    assert set(declared()) <= set(nat.EXPORTED)


def test_abi_version_and_counters():
    lib = nat.lib()
    assert lib.pt_abi_version() == 1
    assert lib.pt_launch_count() >= 0


def test_null_arguments_rejected_without_device():
    lib = nat.lib()
    h = C.c_void_p()
    rc = lib.pt_create(None, None, 0, None, None, None, 0, None, 0, 0, C.byref(h))
    assert rc == nat.PT_EINVAL
    assert b"null" in lib.pt_last_error()
    with pytest.raises(ValueError):
        nat.check(rc)
    assert lib.pt_apply_A(None, None, None, None) == nat.PT_EINVAL
    assert lib.pt_gmres_ws_create(0, 10, 0, C.byref(h)) == nat.PT_EINVAL


def test_struct_layouts_match_header():
    assert C.sizeof(nat.Entry) == 56
    assert C.sizeof(nat.Leaf) == 64
    assert C.sizeof(nat.Layout) == 24
    assert C.sizeof(nat.GmresConfigC) == 16


def test_checked_build_exports_the_same_boundary():
    """libpt_b200_check.so (the executor with invariant asserts and spin-loop
    watchdogs, the stand-in for compute-sanitizer on this pool) exports every
    declared symbol and reports itself as checked; the release build does not."""
    path = nat.LIB_PATH.with_name("libpt_b200_check.so")
    if not path.exists():
        pytest.skip("checked build not built (make -C paper_1410_5910_b200/csrc check)")
    chk = C.CDLL(str(path))
    missing = [n for n in declared() if not hasattr(chk, n)]
    assert not missing, missing
    chk.pt_checked_build.restype = C.c_int32
    assert chk.pt_checked_build() == 1
    assert nat.lib().pt_checked_build() == 0
