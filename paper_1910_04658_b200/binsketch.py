"""Thin ctypes binding over libbinsketch.so (include/binsketch.h).

Argument marshalling only: every step of the hot path runs in the CUDA
kernels behind the C ABI. Tensors must be CUDA tensors of the documented
dtype; calls enqueue on ``torch.cuda.current_stream()``. There is no CPU
fallback: if the library is missing or a call fails, a ``BinSketchError`` is
raised.
"""
from __future__ import annotations

import ctypes
import os

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("BINSKETCH_LIB_VARIANT") or os.path.join(_HERE, "libbinsketch.so")   # variant: dev A/B builds only

IP, HAM, JS, COS = 1, 2, 4, 8
MEASURES = {"ip": IP, "ham": HAM, "js": JS, "cos": COS}
TOPK_EXCLUDE_SELF = 1
MAX_K = 256
OP_ANDPOPC, OP_ESTIMATE, OP_TOPK, OP_JOIN, OP_JOIN_LIST, OP_BCS_ESTIMATE, OP_MSE = 1, 2, 3, 4, 5, 6, 7
MSE_BCS = 1
JOIN_EXCLUDE_SELF, JOIN_EXACT = 1, 2
MAX_THRESHOLDS = 16

STATUS = {0: "OK", 1: "EINVAL", 2: "EINDEX", 3: "ECUDA", 4: "EWORKSPACE", 5: "EUNSUPPORTED"}

# name -> (restype, argtypes)
_u32, _u64, _i32, _vp, _dbl, _sz, _int = (ctypes.c_uint32, ctypes.c_uint64, ctypes.c_int32, ctypes.c_void_p,
                                          ctypes.c_double, ctypes.c_size_t, ctypes.c_int)
SIGNATURES = {
    "binsketch_words": (_u32, [_u32]),
    "binsketch_recommended_N": (_u32, [_u32, _dbl]),
    "binsketch_make_pi": (_int, [_u64, _u64, _u32, _vp, _vp]),
    "binsketch_build": (_int, [_vp, _u64, _u32, _vp, _vp, _u64, _vp, _vp]),
    "binsketch_build_seeded": (_int, [_u64, _u64, _u32, _vp, _vp, _u64, _vp, _vp]),
    "binsketch_bcs_build": (_int, [_vp, _u64, _u32, _vp, _vp, _u64, _vp, _vp]),
    "binsketch_bcs_build_seeded": (_int, [_u64, _u64, _u32, _vp, _vp, _u64, _vp, _vp]),
    "binsketch_bcs_estimate": (_int, [_vp, _u64, _vp, _u64, _u32, _u64, _u32, _vp, _vp, _sz, _vp]),
    "binsketch_bcs_table": (_int, [_u32, _u64, _vp]),
    "binsketch_popcount": (_int, [_vp, _u64, _u32, _vp, _vp]),
    "binsketch_andpopc": (_int, [_vp, _u64, _vp, _u64, _u32, _vp, _vp, _sz, _vp]),
    "binsketch_estimate": (_int, [_vp, _u64, _vp, _u64, _u32, _u64, _u32, _vp, _vp, _sz, _vp]),
    "binsketch_topk": (_int, [_vp, _u64, _vp, _u64, _u32, _u64, _u32, _u32, _u32, _vp, _vp, _vp, _sz, _vp]),
    "binsketch_join": (_int, [_vp, _u64, _vp, _u64, _u32, _u64, _u32, _vp, _u32, _u32, _vp, _vp, _sz, _vp]),
    "binsketch_join_list": (_int, [_vp, _vp, _u64, _vp, _u64, _u32, _u64, _u32, _u32, _vp, _vp, _vp, _u64, _vp, _sz,
                                   _vp]),
    "binsketch_join_confusion": (_int, [_vp, _vp, _u64, _u64, _vp, _vp]),
    "binsketch_mse": (_int, [_vp, _vp, _u64, _u32, _u64, _u32, _vp, _u32, _u32, _vp, _vp, _vp, _sz, _vp]),
    "binsketch_onehot": (_int, [_vp, _u64, _u32, _vp, _vp, _vp, _vp]),
    "binsketch_categorical_estimate": (_int, [_vp, _u64, _vp, _u64, _u32, _u64, _vp, _vp, _sz, _vp]),
    "binsketch_workspace_bytes": (_sz, [_int, _u64, _u64, _u32, _u32]),
    "binsketch_topk_path": (_int, [_u64, _u64, _u32, _u64, _u32]),
    "binsketch_card_table": (_int, [_u32, _u64, _vp]),
    "binsketch_device_status": (_int, [_vp]),
    "binsketch_launch_count": (_u64, []),
    "binsketch_strerror": (ctypes.c_char_p, [_int]),
}


class BinSketchError(RuntimeError):
    def __init__(self, fn: str, code: int):
        self.code = code
        msg = _lib().binsketch_strerror(code).decode() if _LIB is not None else STATUS.get(code, "?")
        super().__init__(f"{fn}: {STATUS.get(code, code)} ({msg})")


_LIB = None


def _lib():
    global _LIB
    if _LIB is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} not built: run `python -m paper_1910_04658_b200.buildlib` "
                              "(there is no CPU fallback)")
        lib = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            f = getattr(lib, name)
            f.restype = res
            f.argtypes = args
        _LIB = lib
    return _LIB


def _check(fn: str, code: int):
    if code != 0:
        raise BinSketchError(fn, code)


def _stream():
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def _dev(t: torch.Tensor, dtype: torch.dtype, name: str):
    if not isinstance(t, torch.Tensor) or not t.is_cuda:
        raise TypeError(f"{name} must be a CUDA tensor")
    if t.dtype != dtype:
        raise TypeError(f"{name} must be {dtype}, got {t.dtype}")
    if not t.is_contiguous():
        raise ValueError(f"{name} must be contiguous")
    return ctypes.c_void_p(t.data_ptr())


def _words_tensor(t, name):
    if t.dtype not in (torch.int32, torch.uint32):
        raise TypeError(f"{name} must hold uint32 sketch words (torch.int32/uint32)")
    return _dev(t, t.dtype, name)


# ------------------------------------------------------------------ API ---
def words(N: int) -> int:
    return int(_lib().binsketch_words(N))


def recommended_N(psi: int, rho: float) -> int:
    return int(_lib().binsketch_recommended_N(psi, rho))


def make_pi(seed: int, d: int, N: int, out: torch.Tensor | None = None) -> torch.Tensor:
    if out is None:
        out = torch.empty(d, dtype=torch.int32, device="cuda")
    _check("binsketch_make_pi", _lib().binsketch_make_pi(seed, d, N, _words_tensor(out, "pi") if d else None, _stream()))
    return out


def build(pi: torch.Tensor, d: int, N: int, indptr: torch.Tensor, indices: torch.Tensor,
          out: torch.Tensor | None = None) -> torch.Tensor:
    n = indptr.numel() - 1
    if out is None:
        out = torch.empty((n, words(N)), dtype=torch.int32, device="cuda")
    _check("binsketch_build", _lib().binsketch_build(
        _words_tensor(pi, "pi") if pi.numel() else None, d, N, _dev(indptr, torch.int64, "indptr"),
        _dev(indices, torch.int32, "indices") if indices.numel() else None, n,
        _words_tensor(out, "out") if out.numel() else None, _stream()))
    return out


def build_seeded(seed: int, d: int, N: int, indptr: torch.Tensor, indices: torch.Tensor,
                 out: torch.Tensor | None = None) -> torch.Tensor:
    n = indptr.numel() - 1
    if out is None:
        out = torch.empty((n, words(N)), dtype=torch.int32, device="cuda")
    _check("binsketch_build_seeded", _lib().binsketch_build_seeded(
        seed, d, N, _dev(indptr, torch.int64, "indptr"),
        _dev(indices, torch.int32, "indices") if indices.numel() else None, n,
        _words_tensor(out, "out") if out.numel() else None, _stream()))
    return out


def bcs_build(pi: torch.Tensor, d: int, N: int, indptr: torch.Tensor, indices: torch.Tensor,
              out: torch.Tensor | None = None) -> torch.Tensor:
    """BCS parity sketches with a pi table."""
    n = indptr.numel() - 1
    if out is None:
        out = torch.empty((n, words(N)), dtype=torch.int32, device="cuda")
    _check("binsketch_bcs_build", _lib().binsketch_bcs_build(
        _words_tensor(pi, "pi") if pi.numel() else None, d, N, _dev(indptr, torch.int64, "indptr"),
        _dev(indices, torch.int32, "indices") if indices.numel() else None, n,
        _words_tensor(out, "out") if out.numel() else None, _stream()))
    return out


def bcs_build_seeded(seed: int, d: int, N: int, indptr: torch.Tensor, indices: torch.Tensor,
                     out: torch.Tensor | None = None) -> torch.Tensor:
    n = indptr.numel() - 1
    if out is None:
        out = torch.empty((n, words(N)), dtype=torch.int32, device="cuda")
    _check("binsketch_bcs_build_seeded", _lib().binsketch_bcs_build_seeded(
        seed, d, N, _dev(indptr, torch.int64, "indptr"),
        _dev(indices, torch.int32, "indices") if indices.numel() else None, n,
        _words_tensor(out, "out") if out.numel() else None, _stream()))
    return out


def bcs_estimate(A: torch.Tensor, B: torch.Tensor, N: int, d: int, measure: int = 15,
                 out: torch.Tensor | None = None, ws=None) -> torch.Tensor:
    na, nb = A.shape[0], B.shape[0]
    planes = bin(measure & 15).count("1")
    if out is None:
        out = torch.empty((planes, na, nb), dtype=torch.float32, device="cuda")
    ws, wp, wn = _workspace(OP_BCS_ESTIMATE, na, nb, N, 0, ws)
    _check("binsketch_bcs_estimate", _lib().binsketch_bcs_estimate(
        _words_tensor(A, "A") if na else None, na, _words_tensor(B, "B") if nb else None, nb, N, d, measure,
        _dev(out, torch.float32, "out") if out.numel() else None, wp, wn, _stream()))
    return out


def bcs_table(N: int, d: int):
    import numpy as np
    out = np.empty(N + 1, dtype=np.float64)
    _check("binsketch_bcs_table", _lib().binsketch_bcs_table(N, d, out.ctypes.data))
    return out


def popcount(sk: torch.Tensor, N: int, out: torch.Tensor | None = None) -> torch.Tensor:
    n = sk.shape[0]
    if out is None:
        out = torch.empty(n, dtype=torch.int32, device="cuda")
    _check("binsketch_popcount", _lib().binsketch_popcount(
        _words_tensor(sk, "sk") if n else None, n, N, _dev(out, torch.int32, "out") if n else None, _stream()))
    return out


def workspace_bytes(op: int, na: int, nb: int, N: int, k: int = 0) -> int:
    return int(_lib().binsketch_workspace_bytes(op, na, nb, N, k))


PATH_NAMES = {0: "none", 1: "tc_fused", 2: "tc_screen", 3: "tc_pab", 4: "cuda"}


def topk_path(nq: int, ndb: int, N: int, d: int, k: int) -> str:
    """The kernel path binsketch_topk takes for these sizes (host-only query)."""
    return PATH_NAMES[int(_lib().binsketch_topk_path(nq, ndb, N, d, k))]


def _workspace(op, na, nb, N, k, ws):
    need = workspace_bytes(op, na, nb, N, k)
    if ws is None:
        ws = torch.empty(max(need, 1), dtype=torch.uint8, device="cuda")
    return ws, ctypes.c_void_p(ws.data_ptr()), ws.numel()


def andpopc(A: torch.Tensor, B: torch.Tensor, N: int, out: torch.Tensor | None = None, ws=None) -> torch.Tensor:
    na, nb = A.shape[0], B.shape[0]
    if out is None:
        out = torch.empty((na, nb), dtype=torch.int32, device="cuda")
    ws, wp, wn = _workspace(OP_ANDPOPC, na, nb, N, 0, ws)
    _check("binsketch_andpopc", _lib().binsketch_andpopc(
        _words_tensor(A, "A") if na else None, na, _words_tensor(B, "B") if nb else None, nb, N,
        _dev(out, torch.int32, "out") if out.numel() else None, wp, wn, _stream()))
    return out


def estimate(A: torch.Tensor, B: torch.Tensor, N: int, d: int, measure: int = 15,
             out: torch.Tensor | None = None, ws=None) -> torch.Tensor:
    na, nb = A.shape[0], B.shape[0]
    planes = bin(measure & 15).count("1")
    if out is None:
        out = torch.empty((planes, na, nb), dtype=torch.float32, device="cuda")
    ws, wp, wn = _workspace(OP_ESTIMATE, na, nb, N, 0, ws)
    _check("binsketch_estimate", _lib().binsketch_estimate(
        _words_tensor(A, "A") if na else None, na, _words_tensor(B, "B") if nb else None, nb, N, d, measure,
        _dev(out, torch.float32, "out") if out.numel() else None, wp, wn, _stream()))
    return out


def topk(Q: torch.Tensor, D: torch.Tensor, N: int, d: int, measure: int, k: int, exclude_self: bool = False,
         out_idx: torch.Tensor | None = None, out_score: torch.Tensor | None = None, ws=None):
    nq, ndb = Q.shape[0], D.shape[0]
    planes = bin(measure & 15).count("1")   # several measures: lists stacked [measure][nq][k]
    shape = (nq, k) if planes == 1 else (planes, nq, k)
    if out_idx is None:
        out_idx = torch.empty(shape, dtype=torch.int32, device="cuda")
    if out_score is None:
        out_score = torch.empty(shape, dtype=torch.float32, device="cuda")
    ws, wp, wn = _workspace(OP_TOPK, nq, ndb, N, k, ws)
    _check("binsketch_topk", _lib().binsketch_topk(
        _words_tensor(Q, "queries") if nq else None, nq, _words_tensor(D, "db") if ndb else None, ndb, N, d,
        measure, k, TOPK_EXCLUDE_SELF if exclude_self else 0,
        _dev(out_idx, torch.int32, "out_idx") if out_idx.numel() else None,
        _dev(out_score, torch.float32, "out_score") if out_score.numel() else None, wp, wn, _stream()))
    return out_idx, out_score


def join(Q: torch.Tensor, D: torch.Tensor, N: int, d: int, measure: int, thresholds, exclude_self: bool = False,
         exact: bool = False, out: torch.Tensor | None = None, ws=None) -> torch.Tensor:
    """Threshold join (Exp. 2): int32 bit planes [nthr][nq][ceil(ndb/32)] (binsketch_join)."""
    nq, ndb = Q.shape[0], D.shape[0]
    thr = (ctypes.c_double * len(thresholds))(*[float(t) for t in thresholds])
    wpr = (ndb + 31) // 32
    if out is None:
        out = torch.empty((len(thresholds), nq, wpr), dtype=torch.int32, device="cuda")
    ws, wp, wn = _workspace(OP_JOIN, nq, ndb, N, 0, ws)
    flags = (JOIN_EXCLUDE_SELF if exclude_self else 0) | (JOIN_EXACT if exact else 0)
    _check("binsketch_join", _lib().binsketch_join(
        _words_tensor(Q, "queries") if nq else None, nq, _words_tensor(D, "db") if ndb else None, ndb, N, d, measure,
        ctypes.cast(thr, ctypes.c_void_p), len(thresholds), flags,
        _words_tensor(out, "out_bits") if out.numel() else None, wp, wn, _stream()))
    return out


def join_list(bits: torch.Tensor, Q: torch.Tensor, D: torch.Tensor, N: int, d: int, measure: int,
              exact: bool = False, ws=None):
    """CSR match list of one join plane: (row_ptr int64[nq+1], cols int32[total], scores float[total])."""
    nq, ndb = Q.shape[0], D.shape[0]
    row_ptr = torch.empty(nq + 1, dtype=torch.int64, device="cuda")
    ws, wp, wn = _workspace(OP_JOIN_LIST, nq, ndb, N, 0, ws)
    flags = JOIN_EXACT if exact else 0
    args = lambda cap, oj, osc: _lib().binsketch_join_list(   # noqa: E731
        _words_tensor(bits, "bits") if bits.numel() else None, _words_tensor(Q, "queries") if nq else None, nq,
        _words_tensor(D, "db") if ndb else None, ndb, N, d, measure, flags, _dev(row_ptr, torch.int64, "row_ptr"),
        oj, osc, cap, wp, wn, _stream())
    if nq == 0:
        row_ptr.zero_()
        return row_ptr, torch.empty(0, dtype=torch.int32, device="cuda"), torch.empty(0, device="cuda")
    _check("binsketch_join_list", args(0, None, None))
    total = int(row_ptr[-1].item())
    cols = torch.empty(max(total, 1), dtype=torch.int32, device="cuda")
    scores = torch.empty(max(total, 1), dtype=torch.float32, device="cuda")
    if total:
        _check("binsketch_join_list", args(total, _dev(cols, torch.int32, "out_j"), _dev(scores, torch.float32,
                                                                                         "out_score")))
    return row_ptr, cols[:total], scores[:total]


def join_confusion(bits_est: torch.Tensor, bits_true: torch.Tensor, ndb: int) -> torch.Tensor:
    """int64 [3][nq]: |O'|, |O|, |O' ∩ O| per query (binsketch_join_confusion)."""
    nq = bits_est.shape[0]
    out = torch.empty((3, nq), dtype=torch.int64, device="cuda")
    if nq:
        _check("binsketch_join_confusion", _lib().binsketch_join_confusion(
            _words_tensor(bits_est, "bits_est") if bits_est.numel() else None,
            _words_tensor(bits_true, "bits_true") if bits_true.numel() else None, nq, ndb,
            _dev(out, torch.int64, "out"), _stream()))
    return out


def mse(S: torch.Tensor, X: torch.Tensor, N: int, d: int, measure: int, thresholds, bcs: bool = False, ws=None):
    """Experiment 1 sums (binsketch_mse): device (sse float64[nthr], count int64[nthr])."""
    n = S.shape[0]
    thr = (ctypes.c_double * len(thresholds))(*[float(t) for t in thresholds])
    sse = torch.empty(len(thresholds), dtype=torch.float64, device="cuda")
    cnt = torch.empty(len(thresholds), dtype=torch.int64, device="cuda")
    ws, wp, wn = _workspace(OP_MSE, n, d, N, 0, ws)
    _check("binsketch_mse", _lib().binsketch_mse(
        _words_tensor(S, "sketches") if n else None, _words_tensor(X, "exact") if n else None, n, N, d, measure,
        ctypes.cast(thr, ctypes.c_void_p), len(thresholds), MSE_BCS if bcs else 0,
        _dev(sse, torch.float64, "out_sse"), _dev(cnt, torch.int64, "out_count"), wp, wn, _stream()))
    return sse, cnt


def onehot(codes: torch.Tensor, offsets: torch.Tensor):
    """Categorical extension (binsketch_onehot): label codes int32 [n][c] + offsets int64 [c+1]
    (device) -> one-hot CSR (indptr int64 [n+1], indices int32 [n*c])."""
    n, c = codes.shape
    indptr = torch.empty(n + 1, dtype=torch.int64, device="cuda")
    indices = torch.empty(n * c, dtype=torch.int32, device="cuda")
    _check("binsketch_onehot", _lib().binsketch_onehot(
        _dev(codes, torch.int32, "codes") if codes.numel() else None, n, c,
        _dev(offsets, torch.int64, "offsets") if c else None, _dev(indptr, torch.int64, "indptr"),
        _dev(indices, torch.int32, "indices") if indices.numel() else None, _stream()))
    return indptr, indices


def categorical_estimate(A: torch.Tensor, B: torch.Tensor, N: int, d: int, out: torch.Tensor | None = None,
                         ws=None) -> torch.Tensor:
    """Estimated categorical distance HAM^/2 (binsketch_categorical_estimate): float [na][nb]."""
    na, nb = A.shape[0], B.shape[0]
    if out is None:
        out = torch.empty((na, nb), dtype=torch.float32, device="cuda")
    ws, wp, wn = _workspace(OP_BCS_ESTIMATE, na, nb, N, 0, ws)
    _check("binsketch_categorical_estimate", _lib().binsketch_categorical_estimate(
        _words_tensor(A, "A") if na else None, na, _words_tensor(B, "B") if nb else None, nb, N, d,
        _dev(out, torch.float32, "out") if out.numel() else None, wp, wn, _stream()))
    return out


def card_table(N: int, d: int):
    import numpy as np
    out = np.empty(N + 1, dtype=np.float64)
    _check("binsketch_card_table", _lib().binsketch_card_table(N, d, out.ctypes.data))
    return out


def launch_count() -> int:
    """Kernels libbinsketch has enqueued since load (for the bench's gpu_launches)."""
    return int(_lib().binsketch_launch_count())


def device_status() -> int:
    """Synchronises the current stream; raises BinSketchError on a latched device error."""
    code = _lib().binsketch_device_status(_stream())
    _check("binsketch_device_status", code)
    return code


# ------------------------------------------------ end-to-end (host buffers) --
def rank_from_host_csr(indptr_h: torch.Tensor, indices_h: torch.Tensor, pi_h: torch.Tensor, d: int, N: int,
                       measure: int, k: int, nq: int | None = None, exclude_self: bool = False,
                       bufs: dict | None = None):
    """The whole path from HOST (pinned) CSR to HOST top-k lists, through the C ABI.

    H2D copy of CSR + pi -> binsketch_build -> binsketch_topk (rows [0,nq) as
    queries against all rows) -> D2H copy of (idx, score). ``bufs`` caches the
    device buffers between calls (so repeated calls do not allocate).
    Returns (out_idx_host, out_score_host, h2d_bytes, d2h_bytes).
    """
    n = indptr_h.numel() - 1
    nq = n if nq is None else nq
    b = bufs if bufs is not None else {}
    if "indptr" not in b:
        b["indptr"] = torch.empty_like(indptr_h, device="cuda")
        b["indices"] = torch.empty_like(indices_h, device="cuda")
        b["pi"] = torch.empty_like(pi_h, device="cuda")
        b["sk"] = torch.empty((n, words(N)), dtype=torch.int32, device="cuda")
        b["idx"] = torch.empty((nq, k), dtype=torch.int32, device="cuda")
        b["score"] = torch.empty((nq, k), dtype=torch.float32, device="cuda")
        b["ws"] = torch.empty(max(1, workspace_bytes(OP_TOPK, nq, n, N, k)), dtype=torch.uint8, device="cuda")
        b["idx_h"] = torch.empty((nq, k), dtype=torch.int32, pin_memory=True)
        b["score_h"] = torch.empty((nq, k), dtype=torch.float32, pin_memory=True)
    b["indptr"].copy_(indptr_h, non_blocking=True)
    b["indices"].copy_(indices_h, non_blocking=True)
    b["pi"].copy_(pi_h, non_blocking=True)
    build(b["pi"], d, N, b["indptr"], b["indices"], out=b["sk"])
    topk(b["sk"][:nq], b["sk"], N, d, measure, k, exclude_self=exclude_self, out_idx=b["idx"],
         out_score=b["score"], ws=b["ws"])
    b["idx_h"].copy_(b["idx"], non_blocking=True)
    b["score_h"].copy_(b["score"], non_blocking=True)
    h2d = indptr_h.numel() * 8 + indices_h.numel() * 4 + pi_h.numel() * 4
    d2h = nq * k * 8
    return b["idx_h"], b["score_h"], h2d, d2h


def topk_from_host_csr(db_indptr_h: torch.Tensor, db_indices_h: torch.Tensor, pi_h: torch.Tensor, d: int, N: int,
                       measures, k: int, q_indptr_h: torch.Tensor | None = None,
                       q_indices_h: torch.Tensor | None = None, exclude_self: bool = False,
                       bufs: dict | None = None):
    """Host (pinned) CSR in, host top-k lists out, through the C ABI: H2D of the db CSR (and of a
    separate query CSR, if given) and pi -> binsketch_build -> binsketch_topk per measure -> D2H of
    every (idx, score) list. Without a query CSR the db rows are the queries (self-join).
    `measures` (an int bit mask or an iterable of measure bits) is deduplicated; with several
    measures the output planes are stacked in bit order IP, HAM, JS, COS (as binsketch_topk
    writes them), whatever order the caller listed them in.
    Returns ((idx_host, score_host) — [measure][nq][k] for several measures —, h2d_bytes, d2h_bytes)."""
    b = bufs if bufs is not None else {}
    n = db_indptr_h.numel() - 1
    sep = q_indptr_h is not None
    nq = (q_indptr_h.numel() - 1) if sep else n
    bits = measures if isinstance(measures, int) else 0
    if not isinstance(measures, int):
        for m in measures:
            bits |= int(m)
    ms = [m for m in (IP, HAM, JS, COS) if bits & m]
    if "db_ip" not in b:
        b["db_ip"] = torch.empty_like(db_indptr_h, device="cuda")
        b["db_ix"] = torch.empty_like(db_indices_h, device="cuda")
        b["pi"] = torch.empty_like(pi_h, device="cuda")
        b["db_sk"] = torch.empty((n, words(N)), dtype=torch.int32, device="cuda")
        if sep:
            b["q_ip"] = torch.empty_like(q_indptr_h, device="cuda")
            b["q_ix"] = torch.empty_like(q_indices_h, device="cuda")
            b["q_sk"] = torch.empty((nq, words(N)), dtype=torch.int32, device="cuda")
        b["ws"] = torch.empty(max(1, workspace_bytes(OP_TOPK, nq, n, N, k)), dtype=torch.uint8, device="cuda")
        shape = (nq, k) if len(ms) == 1 else (len(ms), nq, k)
        b["out"] = (torch.empty(shape, dtype=torch.int32, device="cuda"),
                    torch.empty(shape, dtype=torch.float32, device="cuda"))
        b["out_h"] = (torch.empty(shape, dtype=torch.int32, pin_memory=True),
                      torch.empty(shape, dtype=torch.float32, pin_memory=True))
    b["db_ip"].copy_(db_indptr_h, non_blocking=True)
    b["db_ix"].copy_(db_indices_h, non_blocking=True)
    b["pi"].copy_(pi_h, non_blocking=True)
    h2d = db_indptr_h.numel() * 8 + db_indices_h.numel() * 4 + pi_h.numel() * 4
    build(b["pi"], d, N, b["db_ip"], b["db_ix"], out=b["db_sk"])
    if sep:
        b["q_ip"].copy_(q_indptr_h, non_blocking=True)
        b["q_ix"].copy_(q_indices_h, non_blocking=True)
        h2d += q_indptr_h.numel() * 8 + q_indices_h.numel() * 4
        build(b["pi"], d, N, b["q_ip"], b["q_ix"], out=b["q_sk"])
    qs = b["q_sk"] if sep else b["db_sk"]
    mask = 0
    for m in ms:
        mask |= m
    (oi, osc), (hi, hs) = b["out"], b["out_h"]
    topk(qs, b["db_sk"], N, d, mask, k, exclude_self=exclude_self, out_idx=oi, out_score=osc, ws=b["ws"])
    hi.copy_(oi, non_blocking=True)
    hs.copy_(osc, non_blocking=True)
    d2h = len(ms) * nq * k * 8
    return b["out_h"], h2d, d2h


def topk_from_host_csr_batches(batches, pi_h: torch.Tensor, d: int, N: int, measures, k: int,
                               exclude_self: bool = False, bufs: dict | None = None, on_result=None,
                               before_batch=None):
    """Streaming form of `topk_from_host_csr` over a sequence of host (pinned) CSR batches: each batch
    is (db_indptr, db_indices) — a self-join — or (db_indptr, db_indices, q_indptr, q_indices). Batch
    i+1's H2D copies run on a copy stream while batch i is built and searched, and batch i's lists are
    copied back while batch i+1 computes (one device CSR buffer per side, released by an event after
    each build; two device + two pinned output buffers). Every batch still copies its own inputs in
    and its own lists out. `before_batch(i)` (optional) is enqueued on the compute stream before batch
    i's build; `on_result(i, (idx_h, score_h))` is called once batch i's lists are on the host (the
    pinned buffers are reused two batches later). Returns (h2d_bytes, d2h_bytes) of the last batch."""
    b = bufs if bufs is not None else {}
    bits = measures if isinstance(measures, int) else 0
    if not isinstance(measures, int):
        for m in measures:
            bits |= int(m)
    ms = [m for m in (IP, HAM, JS, COS) if bits & m]
    mask = 0
    for m in ms:
        mask |= m
    comp = torch.cuda.current_stream()
    if "copy" not in b:
        b["copy"] = torch.cuda.Stream()
    copy = b["copy"]
    batches = [tuple(x) for x in batches]
    sep = len(batches[0]) == 4
    n = batches[0][0].numel() - 1
    nq = (batches[0][2].numel() - 1) if sep else n
    if b.get("shape") != (n, nq, sep):
        b["shape"] = (n, nq, sep)
        b["dev"] = [None] * 4
        b["pi"] = torch.empty_like(pi_h, device="cuda")
        b["sk"] = torch.empty((n, words(N)), dtype=torch.int32, device="cuda")
        b["qsk"] = torch.empty((nq, words(N)), dtype=torch.int32, device="cuda") if sep else b["sk"]
        b["ws"] = torch.empty(max(1, workspace_bytes(OP_TOPK, nq, n, N, k)), dtype=torch.uint8, device="cuda")
        shape = (nq, k) if len(ms) == 1 else (len(ms), nq, k)
        b["out"] = [(torch.empty(shape, dtype=torch.int32, device="cuda"),
                     torch.empty(shape, dtype=torch.float32, device="cuda")) for _ in range(2)]
        b["out_h"] = [(torch.empty(shape, dtype=torch.int32, pin_memory=True),
                       torch.empty(shape, dtype=torch.float32, pin_memory=True)) for _ in range(2)]
    for j, t in enumerate(batches[0]):                 # device CSR buffers sized for the largest batch
        need = max(x[j].numel() for x in batches)
        if b["dev"][j] is None or b["dev"][j].numel() < need:
            b["dev"][j] = torch.empty(need, dtype=t.dtype, device="cuda")

    def h2d_batch(i):
        with torch.cuda.stream(copy):
            if i == 0:
                copy.wait_stream(comp)                 # after everything already queued on the caller's stream
            else:
                copy.wait_event(b["built"])            # batch i-1's builds no longer read the CSR buffers
            nbytes = 0
            for j, t in enumerate(batches[i]):
                b["dev"][j][: t.numel()].copy_(t, non_blocking=True)
                nbytes += t.numel() * t.element_size()
            b["pi"].copy_(pi_h, non_blocking=True)
            nbytes += pi_h.numel() * pi_h.element_size()
            ev = torch.cuda.Event()
            ev.record(copy)
        return ev, nbytes

    pend = []
    h2d = d2h = 0
    ev_in, nb_in = h2d_batch(0)
    for i, bt in enumerate(batches):
        if before_batch is not None:
            before_batch(i)
        comp.wait_event(ev_in)
        h2d = nb_in
        ni = bt[0].numel() - 1
        build(b["pi"], d, N, b["dev"][0][: ni + 1], b["dev"][1][: bt[1].numel()], out=b["sk"][:ni])
        if sep:
            nqi = bt[2].numel() - 1
            build(b["pi"], d, N, b["dev"][2][: nqi + 1], b["dev"][3][: bt[3].numel()], out=b["qsk"][:nqi])
        b["built"] = torch.cuda.Event()
        b["built"].record(comp)
        if i + 1 < len(batches):
            ev_in, nb_in = h2d_batch(i + 1)          # overlaps this batch's top-k
        oi, osc = b["out"][i % 2]
        topk(b["qsk"], b["sk"], N, d, mask, k, exclude_self=exclude_self, out_idx=oi, out_score=osc, ws=b["ws"])
        done = torch.cuda.Event()
        done.record(comp)
        hi, hs = b["out_h"][i % 2]
        with torch.cuda.stream(copy):
            copy.wait_event(done)
            hi.copy_(oi, non_blocking=True)
            hs.copy_(osc, non_blocking=True)
            ev_out = torch.cuda.Event()
            ev_out.record(copy)
        d2h = oi.numel() * 4 + osc.numel() * 4
        pend.append((i, ev_out))
        while len(pend) > 1:                         # batch i-1's lists: hand over before its buffers recycle
            j, ev = pend.pop(0)
            ev.synchronize()
            if on_result is not None:
                on_result(j, b["out_h"][j % 2])
    comp.wait_stream(copy)                           # the compute stream now orders after the last lists
    for j, ev in pend:
        ev.synchronize()
        if on_result is not None:
            on_result(j, b["out_h"][j % 2])
    return h2d, d2h
