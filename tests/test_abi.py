"""Host-side checks of the C-ABI library: it loads, exports every symbol include/l1dm.h
declares, and its pure-host calls behave.  No compute calls (no GPU needed)."""
import ctypes
import os
import re

import pytest
import torch

import paper_2210_15114_b200 as l1
from conftest import ROOT


def header_symbols():
    src = open(os.path.join(ROOT, "include", "l1dm.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(l1dm_[a-z0-9_]+)\s*\(", src)))


def test_library_loads_and_exports_every_declared_symbol():
    lib = l1.load_library()
    syms = header_symbols()
    assert len(syms) >= 15
    for s in syms:
        assert hasattr(lib, s), f"libl1dm.so does not export {s}"
    assert set(l1.EXPORTS) <= set(syms)
    assert l1.l1dm_version().startswith("l1dm")


def test_library_is_sm100a():
    out = os.popen(f"cuobjdump --list-elf {l1.LIB_PATH} 2>&1").read()
    assert "sm_100a" in out


def test_null_and_range_arguments_are_rejected_without_a_device():
    lib = l1.load_library()
    h = ctypes.c_void_p()
    assert lib.l1dm_prepare(None, 10, 3, ctypes.byref(h)) == -1
    assert h.value is None
    buf = (ctypes.c_float * 30)()
    assert lib.l1dm_prepare(buf, 0, 3, ctypes.byref(h)) == -1
    assert lib.l1dm_prepare(buf, 10, 0, ctypes.byref(h)) == -1
    assert lib.l1dm_prepare(buf, 1 << 32, 3, ctypes.byref(h)) == -1
    assert lib.l1dm_prepare_ex(buf, 10, 3, 2, 5, None, ctypes.byref(h)) == -1
    assert lib.l1dm_prepare_ex(buf, 10, 3, 2, 2, None, ctypes.byref(h)) == -1
    assert lib.l1dm_matvec(None, buf, 1, buf) == -1
    assert b"NULL" in lib.l1dm_last_error()
    lib.l1dm_free(None)  # no-op


@pytest.mark.skipif(torch.cuda.is_available(), reason="checks the no-device path")
def test_no_cpu_fallback_without_device():
    X = torch.rand(50, 3)
    with pytest.raises(l1.L1dmError) as e:
        l1.l1dm_prepare(X)
    assert e.value.name == "L1DM_EDEVICE"


def test_missing_library_raises_instead_of_falling_back(tmp_path):
    """A fresh interpreter pointed at a library path that does not exist must fail on the
    first call (ImportError), never compute on the CPU."""
    import subprocess
    import sys
    code = ("import torch, paper_2210_15114_b200 as l1\n"
            "try:\n"
            "    l1.l1dm_prepare(torch.rand(8, 2))\n"
            "except ImportError as e:\n"
            "    print('raised', 'no CPU fallback' in str(e))\n")
    env = dict(os.environ, L1DM_LIB=str(tmp_path / "absent.so"))
    out = subprocess.run([sys.executable, "-c", code], cwd=ROOT, env=env, capture_output=True,
                         text=True, timeout=300)
    assert out.stdout.strip() == "raised True", out.stdout + out.stderr[-2000:]


def test_product_package_never_touches_the_oracle():
    """Only tests/, __graft_entry__.smoke() and bench.py's CPU arms may use oracle/: no module
    of the package imports it or names it in a load path."""
    pkg = os.path.join(ROOT, "paper_2210_15114_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if not f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                continue
            src = open(os.path.join(dirpath, f)).read()
            assert not re.search(r"^\s*(import|from)\s+oracle\b", src, flags=re.M), f
            assert not re.search(r"""#\s*include\s*["<][^">]*oracle|["']oracle[/.]""", src), f
