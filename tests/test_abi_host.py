"""C-ABI library, CPU-side checks (no GPU compute).

* libbinsketch.so loads and exports every entry point include/binsketch.h declares;
* host-only entry points (sizing rule, words, strerror, workspace sizing, the
  host-built cardinality table) and host-detectable argument errors;
* the product package shares no code with oracle/ and never imports it.
"""
import ctypes
import math
import os
import re

import numpy as np
import pytest

import oracle
from bsk_helpers import ROOT

from paper_1910_04658_b200 import buildlib as libbuild

HEADER = os.path.join(ROOT, "include", "binsketch.h")


@pytest.fixture(scope="module")
def lib():
    libbuild.build()
    return ctypes.CDLL(libbuild.LIB)


def _declared():
    src = open(HEADER).read()
    return sorted(set(re.findall(r"\b(binsketch_[a-z_N]+)\s*\(", src)))


def test_exports_every_declared_symbol(lib):
    names = _declared()
    assert len(names) == 25
    for name in names:
        assert hasattr(lib, name), name
    from paper_1910_04658_b200.binsketch import SIGNATURES
    assert sorted(SIGNATURES) == names      # the binding wraps exactly the ABI


def test_topk_path_host(lib, monkeypatch):
    """binsketch_topk_path (host-only): the kernel path a top-k call takes — the fused tensor-core
    kernel for the Large shape, the tensor-core screen for Ranking (k = 100), the CUDA-core kernels
    for small calls (nq * ndb <= 2^25), none for empty calls; the engine override wins."""
    from paper_1910_04658_b200 import binsketch as bs
    monkeypatch.setenv("BINSKETCH_TOPK_SMALL", "1")
    monkeypatch.delenv("BINSKETCH_ENGINE", raising=False)
    assert bs.topk_path(200_000, 200_000, 1024, 500_000, 50) == "tc_fused"
    assert bs.topk_path(1000, 100_000, 4096, 102_660, 100) == "tc_screen"
    assert bs.topk_path(1000, 1000, 1224, 5000, 10) == "cuda"
    assert bs.topk_path(0, 1000, 1224, 5000, 10) == "none" and bs.topk_path(10, 10, 1224, 5000, 0) == "none"
    monkeypatch.setenv("BINSKETCH_ENGINE", "tc")
    assert bs.topk_path(1000, 1000, 1224, 5000, 10) == "tc_fused"
    monkeypatch.setenv("BINSKETCH_ENGINE", "cuda")
    assert bs.topk_path(200_000, 200_000, 1024, 500_000, 50) == "cuda"


def test_host_entry_points(lib):
    lib.binsketch_recommended_N.restype = ctypes.c_uint32
    lib.binsketch_recommended_N.argtypes = [ctypes.c_uint32, ctypes.c_double]
    for psi, rho in [(100, 0.1), (20, 0.1), (1, 0.999999), (0, 0.1), (5, 1.5), (300, 0.01)]:
        assert lib.binsketch_recommended_N(psi, rho) == oracle.recommended_N(psi, rho)
    lib.binsketch_words.restype = ctypes.c_uint32
    assert [lib.binsketch_words(N) for N in (2, 32, 33, 1224, 5000)] == [1, 1, 2, 39, 157]
    lib.binsketch_strerror.restype = ctypes.c_char_p
    for code in range(6):
        assert lib.binsketch_strerror(code)


@pytest.mark.parametrize("N,d", [(2, 10), (1000, 28102), (1224, 5000), (2000, 28102), (4096, 102660),
                                 (5000, 28102), (1024, 1 << 20)])
def test_card_table_bit_identical_to_oracle(lib, N, d):
    """binsketch_card_table (host libm log1p) == the oracle's table, byte for byte (R-C3)."""
    lib.binsketch_card_table.argtypes = [ctypes.c_uint32, ctypes.c_uint64, ctypes.c_void_p]
    out = np.empty(N + 1, dtype=np.float64)
    assert lib.binsketch_card_table(N, d, out.ctypes.data) == 0
    assert out.tobytes() == oracle.card_table(N, d).tobytes()


def test_bcs_table_bit_identical_to_oracle(lib):
    lib.binsketch_bcs_table.argtypes = [ctypes.c_uint32, ctypes.c_uint64, ctypes.c_void_p]
    for N, d in ((2, 10), (1024, 50_000), (4096, 102_660), (1223, 5000)):
        out = np.empty(N + 1, dtype=np.float64)
        assert lib.binsketch_bcs_table(N, d, out.ctypes.data) == 0
        assert out.tobytes() == oracle.bcs_table(N, d).tobytes()


def test_workspace_sizing(lib):
    lib.binsketch_workspace_bytes.restype = ctypes.c_size_t
    lib.binsketch_workspace_bytes.argtypes = [ctypes.c_int, ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint32,
                                              ctypes.c_uint32]
    est = lib.binsketch_workspace_bytes(2, 1000, 1000, 1224, 0)
    assert est >= 1225 * 8 + 2000 * 4
    topk_small = lib.binsketch_workspace_bytes(3, 1000, 100_000, 4096, 100)
    assert topk_small > 4097 * 8 + 101_000 * 4         # includes the split-merge buffers
    assert lib.binsketch_workspace_bytes(3, 1000, 100_000, 4096, 100) == topk_small   # pure function


def test_workspace_estimate_paths(lib, monkeypatch):
    """All-pairs estimates: the default tensor-core path holds the int32 pab table (na*nb*4 bytes)
    in the workspace while it fits the 4 GB budget; the fused epilogue (BINSKETCH_EST_PAB=0) and
    tables beyond the budget do not (K10b). The env knob is read at each call."""
    lib.binsketch_workspace_bytes.restype = ctypes.c_size_t
    lib.binsketch_workspace_bytes.argtypes = [ctypes.c_int, ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint32,
                                              ctypes.c_uint32]
    monkeypatch.delenv("BINSKETCH_ENGINE", raising=False)
    monkeypatch.delenv("BINSKETCH_EST_PAB", raising=False)
    na, nb = 10_000, 10_000
    with_table = lib.binsketch_workspace_bytes(2, na, nb, 1000, 0)
    assert with_table >= na * nb * 4
    monkeypatch.setenv("BINSKETCH_EST_PAB", "0")
    fused = lib.binsketch_workspace_bytes(2, na, nb, 1000, 0)
    assert fused < na * nb * 4 and with_table - fused >= na * nb * 4
    monkeypatch.delenv("BINSKETCH_EST_PAB")
    big = lib.binsketch_workspace_bytes(2, 40_000, 40_000, 1000, 0)     # 6.4 GB table: over budget
    assert big < 40_000 * 40_000 * 4
    monkeypatch.setenv("BINSKETCH_ENGINE", "cuda")                       # CUDA-core engine: no table
    assert lib.binsketch_workspace_bytes(2, na, nb, 1000, 0) < na * nb * 4


def test_host_detected_errors(lib):
    vp = ctypes.c_void_p
    lib.binsketch_build.argtypes = [vp, ctypes.c_uint64, ctypes.c_uint32, vp, vp, ctypes.c_uint64, vp, vp]
    lib.binsketch_estimate.argtypes = [vp, ctypes.c_uint64, vp, ctypes.c_uint64, ctypes.c_uint32, ctypes.c_uint64,
                                       ctypes.c_uint32, vp, vp, ctypes.c_size_t, vp]
    lib.binsketch_topk.argtypes = [vp, ctypes.c_uint64, vp, ctypes.c_uint64, ctypes.c_uint32, ctypes.c_uint64,
                                   ctypes.c_uint32, ctypes.c_uint32, ctypes.c_uint32, vp, vp, vp, ctypes.c_size_t, vp]
    lib.binsketch_make_pi.argtypes = [ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint32, vp, vp]
    EINVAL, EUNSUP = 1, 5
    assert lib.binsketch_make_pi(0, 10, 1, None, None) == EINVAL                 # N < 2
    assert lib.binsketch_make_pi(0, 10, 16, None, None) == EINVAL                # null with d > 0
    assert lib.binsketch_build(None, 10, 1, None, None, 5, None, None) == EINVAL  # N < 2
    assert lib.binsketch_build(None, 10, 64, None, None, 5, None, None) == EINVAL  # null pointers
    assert lib.binsketch_build(None, 10, 64, None, None, 0, None, None) == 0      # n = 0: no-op
    assert lib.binsketch_estimate(None, 4, None, 4, 64, 10, 0, None, None, 0, None) == EINVAL   # measure 0
    assert lib.binsketch_estimate(None, 4, None, 4, 64, 10, 16, None, None, 0, None) == EINVAL  # bad bit
    assert lib.binsketch_estimate(None, 0, None, 4, 64, 10, 15, None, None, 0, None) == 0       # empty
    assert lib.binsketch_topk(None, 4, None, 4, 64, 10, 16, 5, 0, None, None, None, 0, None) == EINVAL  # bad bit
    assert lib.binsketch_topk(None, 4, None, 4, 64, 10, 0, 5, 0, None, None, None, 0, None) == EINVAL   # no measure
    assert lib.binsketch_topk(None, 4, None, 4, 64, 10, 1, 5, 2, None, None, None, 0, None) == EINVAL  # flags
    assert lib.binsketch_topk(None, 4, None, 4, 64, 10, 1, 0, 0, None, None, None, 0, None) == 0       # k = 0
    assert lib.binsketch_topk(vp(8), 4, vp(8), 4, 64, 10, 1, 257, 0, vp(8), vp(8), None, 0, None) == EUNSUP
    # threshold join (host checks happen before any device work)
    u64, u32 = ctypes.c_uint64, ctypes.c_uint32
    lib.binsketch_join.argtypes = [vp, u64, vp, u64, u32, u64, u32, vp, u32, u32, vp, vp, ctypes.c_size_t, vp]
    thr = (ctypes.c_double * 17)(*([0.5] * 17))
    nan = (ctypes.c_double * 1)(float("nan"))
    t1 = ctypes.cast(thr, vp)
    assert lib.binsketch_join(vp(8), 4, vp(8), 4, 64, 10, 4, t1, 1, 0, vp(8), vp(8), 0, None) == 4   # EWORKSPACE
    assert lib.binsketch_join(None, 4, None, 4, 64, 10, 5, t1, 1, 0, None, None, 0, None) == EINVAL  # 2 bits
    assert lib.binsketch_join(None, 4, None, 4, 64, 10, 4, t1, 1, 4, None, None, 0, None) == EINVAL  # flags
    assert lib.binsketch_join(None, 4, None, 4, 64, 10, 4, t1, 0, 0, None, None, 0, None) == EINVAL  # nthr 0
    assert lib.binsketch_join(None, 4, None, 4, 64, 10, 4, t1, 17, 0, None, None, 0, None) == EINVAL  # nthr 17
    assert lib.binsketch_join(None, 4, None, 4, 64, 10, 4, None, 1, 0, None, None, 0, None) == EINVAL  # no thr
    assert lib.binsketch_join(None, 4, None, 4, 64, 10, 4, ctypes.cast(nan, vp), 1, 0, None, None, 0,
                              None) == EINVAL                                                     # NaN
    assert lib.binsketch_join(None, 0, None, 4, 64, 10, 4, t1, 16, 0, None, None, 0, None) == 0       # empty
    assert lib.binsketch_join(None, 4, None, 4, 64, 10, 4, t1, 2, 0, None, None, 0, None) == EINVAL   # nulls
    assert lib.binsketch_join(vp(8), 4, vp(8), 4, 64, 0, 4, t1, 2, 0, vp(8), None, 0, None) == EINVAL  # d = 0
    lib.binsketch_join_confusion.argtypes = [vp, vp, u64, u64, vp, vp]
    assert lib.binsketch_join_confusion(None, None, 0, 5, None, None) == 0
    assert lib.binsketch_join_confusion(None, None, 3, 5, vp(8), None) == EINVAL


def test_size_limits(lib):
    """N beyond the documented limits (binsketch.h BINSKETCH_MAX_N_*) is refused on the host with
    EUNSUPPORTED, before any size arithmetic that could wrap."""
    vp, u64, u32 = ctypes.c_void_p, ctypes.c_uint64, ctypes.c_uint32
    EUNSUP = 5
    big_pairs = 0x01000001
    lib.binsketch_make_pi.argtypes = [u64, u64, u32, vp, vp]
    assert lib.binsketch_make_pi(0, 0, 0xFFFFFFFF, None, None) == 0     # construction: every N (d = 0: no-op)
    lib.binsketch_words.restype = u32
    assert lib.binsketch_words(0xFFFFFFFF) == 0x08000000                # no 32-bit wrap
    lib.binsketch_estimate.argtypes = [vp, u64, vp, u64, u32, u64, u32, vp, vp, ctypes.c_size_t, vp]
    assert lib.binsketch_estimate(vp(8), 4, vp(8), 4, big_pairs, 10, 1, vp(8), vp(8), 0, None) == EUNSUP
    lib.binsketch_topk.argtypes = [vp, u64, vp, u64, u32, u64, u32, u32, u32, vp, vp, vp, ctypes.c_size_t, vp]
    assert lib.binsketch_topk(vp(8), 4, vp(8), 4, big_pairs, 10, 1, 5, 0, vp(8), vp(8), vp(8), 0, None) == EUNSUP
    lib.binsketch_card_table.argtypes = [u32, u64, vp]
    dummy = np.empty(1, dtype=np.float64)
    assert lib.binsketch_card_table(big_pairs, 10, dummy.ctypes.data) == EUNSUP
    lib.binsketch_workspace_bytes.restype = ctypes.c_size_t
    lib.binsketch_workspace_bytes.argtypes = [ctypes.c_int, u64, u64, u32, u32]
    assert lib.binsketch_workspace_bytes(2, 10, 10, big_pairs, 0) == 0
    assert lib.binsketch_workspace_bytes(2, 10, 10, 0x01000000, 0) > 0            # the limit itself is accepted


def test_product_shares_no_code_with_oracle():
    pkg = os.path.join(ROOT, "paper_1910_04658_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                src = open(os.path.join(dirpath, f)).read()
                assert not re.search(r"^\s*(import|from)\s+oracle\b", src, re.M), f
                assert "oracle.cpp" not in src and "liboracle" not in src, f
                assert not re.search(r"^\s*(import|from)\s+synth\b", src, re.M), f
    osrc = open(os.path.join(ROOT, "oracle", "oracle.cpp")).read()
    assert "#include \"binsketch.h\"" not in osrc and "bsk_" not in osrc


def test_binding_fails_loudly_without_the_library(tmp_path):
    """No CPU fallback: with the library absent every call raises (here: a fresh interpreter
    pointed at a missing .so), and without a GPU a compute call raises instead of computing."""
    import subprocess
    import sys
    code = ("import os, sys; sys.path.insert(0, %r); os.environ['BINSKETCH_LIB_VARIANT'] = %r\n"
            "from paper_1910_04658_b200 import binsketch as bs\n"
            "try:\n    bs.words(64)\nexcept ImportError as e:\n    print('raised', e)\n") % (ROOT, str(tmp_path / "missing.so"))
    out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=300)
    assert "raised" in out.stdout and "no CPU fallback" in out.stdout


def test_no_cpu_compute_path_in_the_binding():
    """The binding only marshals arguments: it never imports numpy-based compute or the oracle,
    and every public compute function ends in a libbinsketch call."""
    src = open(os.path.join(ROOT, "paper_1910_04658_b200", "binsketch.py")).read()
    assert "import oracle" not in src and "from oracle" not in src
    for name in ("build", "build_seeded", "popcount", "andpopc", "estimate", "topk", "join", "mse",
                 "bcs_build", "bcs_estimate", "onehot", "categorical_estimate"):
        body = src.split(f"\ndef {name}(", 1)[1].split("\ndef ", 1)[0]
        assert "_lib()." in body, name
