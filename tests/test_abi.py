"""C-ABI boundary checks that need no GPU: the library builds/loads for sm_100a and
exports exactly the entry points include/pnce_b200.h declares."""

import ctypes
import os
import re
import subprocess

import pytest

from paper_2206_05506_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "pnce_b200.h")


@pytest.fixture(scope="module")
def built():
    if not os.path.exists(_lib.LIB_PATH):
        import __graft_entry__
        __graft_entry__.build()
    return _lib.lib()


def header_functions():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"\b(pnce_[a-z0-9_]+)\s*\(", text)))


def test_header_matches_binding_table():
    assert header_functions() == sorted(_lib.EXPORTS)


def test_library_exports_every_symbol(built):
    for name in header_functions():
        assert hasattr(built, name), name
    out = subprocess.run(["nm", "-D", "--defined-only", _lib.LIB_PATH], capture_output=True, text=True).stdout
    for name in header_functions():
        assert re.search(rf"\bT {name}\b", out), name


def test_library_is_sm100a(built):
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", _lib.LIB_PATH],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out
    sass = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-sass", _lib.LIB_PATH],
                          capture_output=True, text=True).stdout
    assert "UTCHMMA" in sass and "UTMALDG" in sass and "LDTM" in sass


def test_host_entry_points_without_gpu(built):
    """Host-only entry points work on a CPU box; config errors map to reference classes."""
    assert built.pnce_version() >= 100
    cfg = _lib.CfgStruct(m=1023, c=64, n_t=64, n_r=64, n_batch=8, l=64, degree=10,
                         tap_mask=(1 << 9) | (1 << 2), state=1, dtype=0)
    assert built.pnce_config_check(ctypes.byref(cfg)) == 0
    bad = _lib.CfgStruct(m=1023, c=64, n_t=64, n_r=64, n_batch=16, l=64, degree=10,
                         tap_mask=(1 << 9) | (1 << 2), state=1, dtype=0)
    import paper_2206_05506_b200 as P
    with pytest.raises(P.InvalidConfigError):
        _lib.check(built.pnce_config_check(ctypes.byref(bad)))
    zero = _lib.CfgStruct(m=1023, c=64, n_t=64, n_r=64, n_batch=8, l=64, degree=10,
                          tap_mask=(1 << 9) | (1 << 2), state=0, dtype=0)
    with pytest.raises(P.ZeroStateError):
        _lib.check(built.pnce_config_check(ctypes.byref(zero)))
    assert built.pnce_kernel_launches() == 0


def test_no_library_gemm(built):
    """The synthesiser's body GEMM runs on the library's own tcgen05 kernel (k_synth_gemm):
    no cuBLAS import or dependency is left in libpnce_b200.so."""
    und = subprocess.run(["nm", "-D", "--undefined-only", _lib.LIB_PATH], capture_output=True, text=True).stdout
    assert "cublas" not in und.lower()
    deps = subprocess.run(["ldd", _lib.LIB_PATH], capture_output=True, text=True).stdout
    assert "cublas" not in deps.lower()
