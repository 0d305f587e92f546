"""CPU tests of the boundary: libgfb.so loads, exports every symbol that
include/gfb.h declares, the Python signature table covers the header, and
the error path works without a GPU (no compute calls here)."""
import ctypes as C
import os
import re
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "gfb.h")
LIB = os.path.join(ROOT, "paper_2212_08200_b200", "lib", "libgfb.so")


def declared():
    txt = open(HEADER).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(gfb_[a-z_0-9]+)\s*\(", txt)))


@pytest.fixture(scope="module")
def lib():
    if not os.path.exists(LIB):
        subprocess.run(["make", "-s", "-j4", "-C",
                        os.path.join(ROOT, "paper_2212_08200_b200", "csrc")], check=True)
    return C.CDLL(LIB)


def test_header_declares_the_boundary():
    names = declared()
    for must in ("gfb_sssp", "gfb_graph_upload", "gfb_advance_push", "gfb_advance_pull",
                 "gfb_filter_unique", "gfb_last_error", "gfb_ctx_create"):
        assert must in names


def test_library_exports_every_declared_symbol(lib):
    out = subprocess.run(["nm", "-D", "--defined-only", LIB], capture_output=True, text=True,
                         check=True).stdout
    exported = set(re.findall(r"\sT\s(gfb_\w+)", out))
    missing = [n for n in declared() if n not in exported]
    assert not missing, missing
    for n in declared():
        getattr(lib, n)


def test_python_binding_covers_header():
    from paper_2212_08200_b200 import _lib
    assert sorted(_lib.SIGNATURES) == declared()


def test_library_does_not_link_nccl():
    """NCCL is bound lazily (xmg.cu nccl_api()): a libgfb.so that linked the
    system libnccl.so.2 and was loaded before torch made `import torch` fail
    (torch's bundled NCCL shares the soname and has newer symbols)."""
    out = subprocess.run(["readelf", "-d", LIB], capture_output=True, text=True,
                         check=True).stdout
    assert "libnccl" not in out
    code = ("import ctypes; ctypes.CDLL(%r, mode=ctypes.RTLD_GLOBAL); import torch; "
            "print('ok')" % LIB)
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0 and "ok" in r.stdout, r.stderr[-2000:]


def test_library_is_sm100a(lib):
    out = subprocess.run(["cuobjdump", "--list-elf", LIB], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_error_path_without_gpu(lib):
    """No device here: ctx creation fails with a status + message, no crash."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    lib.gfb_last_error.restype = C.c_char_p
    h = C.c_void_p()
    rc = lib.gfb_ctx_create(0, C.byref(h))
    assert rc != 0
    assert lib.gfb_last_error()
    assert lib.gfb_version() == 1


def test_opts_default(lib):
    from paper_2212_08200_b200 import _lib
    o = _lib.SsspOpts()
    _lib.load().gfb_sssp_opts_default(C.byref(o))
    assert o.struct_size == C.sizeof(_lib.SsspOpts)
    assert o.direction == _lib.DIR_PUSH and o.compute_pred == 1  # algorithms.hpp:40
    assert abs(o.pull_alpha - 1.05) < 1e-6 and o.defer_pct == 0 and o.advance_tile == 0


def test_product_never_references_oracle():
    """The product path must not route through the checker."""
    pkg = os.path.join(ROOT, "paper_2212_08200_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".hpp", ".cpp", ".h")):
                txt = open(os.path.join(dirpath, f)).read()
                assert "oracle" not in txt.replace("oracle/graflow_oracle.c restates", ""), f
