"""The C-ABI library loads and exports every symbol include/ghostx.h declares
(CPU only: no compute calls that need a device)."""

import ctypes
import os
import re
import subprocess

import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(REPO, "include", "ghostx.h")


def declared():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(ghx_[a-z0-9_]+)\s*\(", src)))


def test_header_declares_api():
    names = declared()
    assert "ghx_plan_build_fill_boundary" in names and "ghx_exec_run" in names
    assert len(names) >= 25


def test_library_exports_every_declared_symbol():
    from paper_2403_12179_b200 import _native as N
    lib = ctypes.CDLL(N.LIB_PATH)
    missing = [n for n in declared() if not hasattr(lib, n)]
    assert not missing, missing


def test_binding_covers_header():
    from paper_2403_12179_b200 import _native as N
    assert set(declared()) == set(N.EXPORTED)


def test_library_is_sm100a():
    from paper_2403_12179_b200 import _native as N
    try:
        out = subprocess.run(["cuobjdump", "--list-elf", N.LIB_PATH], capture_output=True, text=True,
                             timeout=60).stdout
    except (FileNotFoundError, subprocess.TimeoutExpired):
        pytest.skip("cuobjdump unavailable")
    assert "sm_100a" in out


def test_errors_are_codes_not_exceptions():
    from paper_2403_12179_b200 import _native as N
    h = ctypes.c_void_p()
    rc = N.lib.ghx_plan_build_fill_boundary(-1, None, None, None, None, None, 0, ctypes.byref(h))
    assert rc == N.GHX_EINVAL
    assert "bad arguments" in N.last_error()
    with pytest.raises(ValueError):
        N.check(rc)
