"""TEST INFRASTRUCTURE ONLY -- ctypes front end of the CPU oracle.

Only tests/, ``__graft_entry__.smoke()`` and bench.py's CPU-baseline leg may
import this module; it is the checker, never the product.  It wraps
``oracle/build/libqsg_oracle.so`` (built by ``oracle/Makefile``) and adds a
numpy restatement of the reference's code construction:

    gb_rows          code.py:194-231  (build_gb, _circulant_columns)
    tanner_arrays    code.py:150-191  (tanner_graph flat arrays)

Decoder configuration objects may be the reference's ``qsagms.DecoderConfig``
or this package's mirror; both expose ``variant``, ``l_max``, ``alpha``,
``gain`` (``alpha_min``/``alpha_max``/``eta_unsat``) and ``vn_mode``.
"""

from __future__ import annotations

import ctypes as C
import math
import os
import subprocess
from dataclasses import dataclass
from types import SimpleNamespace

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "build", "libqsg_oracle.so")
VARIANTS = ("bp4", "ms", "sms", "sagms")
VN_MODES = ("marginal", "additive")

_lib = None


def build() -> str:
    subprocess.run(["make", "-s", "-C", HERE], check=True)
    return LIB_PATH


class _Graph(C.Structure):
    _fields_ = [
        ("n", C.c_int32), ("m", C.c_int32), ("E", C.c_int64),
        ("edge_cn", C.c_void_p), ("edge_vn", C.c_void_p), ("edge_sym", C.c_void_p),
        ("cn_ptr", C.c_void_p), ("vn_order", C.c_void_p), ("vn_ptr", C.c_void_p),
    ]


class _Cfg(C.Structure):
    _fields_ = [
        ("variant", C.c_int32), ("vn_mode", C.c_int32), ("l_max", C.c_int32),
        ("early_stop", C.c_int32), ("alpha", C.c_double), ("alpha_min", C.c_double),
        ("alpha_max", C.c_double), ("eta_unsat", C.c_double),
    ]


class _Trace(C.Structure):
    _fields_ = [("unsat", C.c_void_p), ("vn_msgs", C.c_void_p),
                ("cn_msgs", C.c_void_p), ("counts", C.c_void_p)]


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            build()
        L = C.CDLL(LIB_PATH)
        vp, i32, i64, dbl, u64 = C.c_void_p, C.c_int32, C.c_int64, C.c_double, C.c_uint64
        L.qsgo_sample_errors.argtypes = [i32, dbl, u64, i64, i64, vp]
        L.qsgo_philox4x64_10.argtypes = [vp, vp, vp]
        L.qsgo_syndromes_of.argtypes = [vp, vp, i64, vp]
        for p in ("32", "64"):
            getattr(L, f"qsgo{p}_decode").argtypes = [vp, vp, dbl, vp, i64, vp, vp, vp, vp, i32]
            getattr(L, f"qsgo{p}_frames").argtypes = [vp, vp, dbl, dbl, u64, i64, i64,
                                                      vp, vp, vp, vp, i32]
        L.qsgo_math32_batch.argtypes = [i32, vp, vp, vp, i64]
        L.qsgo_bp4_mags.argtypes = [vp, i32, vp]
        _lib = L
    return _lib


def _ptr(a):
    return None if a is None else a.ctypes.data


# -- code construction (restated from the reference) -------------------------

def gb_rows(ell, a_exps, b_exps):
    """Rows of build_gb (code.py:201-231): list of [(col, sym)] per check."""
    def circ(exps, sign):
        return [sorted((i + sign * e) % ell for e in exps) for i in range(ell)]
    A, Bm = circ(a_exps, 1), circ(b_exps, 1)
    Bt, At = circ(b_exps, -1), circ(a_exps, -1)
    rows = []
    for i in range(ell):
        rows.append([(j, 1) for j in A[i]] + [(ell + j, 1) for j in Bm[i]])
    for i in range(ell):
        rows.append([(j, 2) for j in Bt[i]] + [(ell + j, 2) for j in At[i]])
    return rows


def tanner_arrays(n, rows):
    """Flat TannerGraph arrays (code.py:150-191) from sparse rows."""
    edge_cn, edge_vn, edge_sym = [], [], []
    vn_adj = [[] for _ in range(n)]
    for i, row in enumerate(rows):
        for j, s in row:
            vn_adj[j].append(len(edge_cn))
            edge_cn.append(i)
            edge_vn.append(j)
            edge_sym.append(s)
    E = len(edge_cn)
    cn_deg = np.array([len(r) for r in rows], dtype=np.int64)
    vn_deg = np.array([len(a) for a in vn_adj], dtype=np.int64)
    vn_order = np.array([e for a in vn_adj for e in a], dtype=np.int64)
    vn_inverse = np.empty(E, dtype=np.int64)
    vn_inverse[vn_order] = np.arange(E)
    return SimpleNamespace(
        n=n, m=len(rows), edge_count=E,
        edges=list(zip(edge_cn, edge_vn, edge_sym)),
        edge_cn=np.array(edge_cn, dtype=np.int64), edge_vn=np.array(edge_vn, dtype=np.int64),
        edge_sym=np.array(edge_sym, dtype=np.uint8),
        cn_ptr=np.concatenate(([0], np.cumsum(cn_deg))).astype(np.int64),
        vn_order=vn_order, vn_inverse=vn_inverse,
        vn_ptr=np.concatenate(([0], np.cumsum(vn_deg))).astype(np.int64),
        cn_degrees=cn_deg, vn_degrees=vn_deg, rows=rows,
    )


def gb_graph(ell, a_exps, b_exps):
    return tanner_arrays(2 * ell, gb_rows(ell, a_exps, b_exps))


# -- the restated hot path ------------------------------------------------------

class Graph:
    """Holds contiguous int64/uint8 copies and the C struct for one graph."""

    def __init__(self, g):
        self.n, self.m = int(g.n), int(g.m)
        self.edge_cn = np.ascontiguousarray(g.edge_cn, dtype=np.int64)
        self.edge_vn = np.ascontiguousarray(g.edge_vn, dtype=np.int64)
        self.edge_sym = np.ascontiguousarray(g.edge_sym, dtype=np.uint8)
        self.cn_ptr = np.ascontiguousarray(g.cn_ptr, dtype=np.int64)
        self.vn_order = np.ascontiguousarray(g.vn_order, dtype=np.int64)
        self.vn_ptr = np.ascontiguousarray(g.vn_ptr, dtype=np.int64)
        self.E = int(self.edge_cn.shape[0])
        self.c = _Graph(self.n, self.m, self.E, _ptr(self.edge_cn), _ptr(self.edge_vn),
                        _ptr(self.edge_sym), _ptr(self.cn_ptr), _ptr(self.vn_order),
                        _ptr(self.vn_ptr))


def _as_graph(g):
    return g if isinstance(g, Graph) else Graph(g)


def _cfg(cfg, early_stop=True):
    gain = getattr(cfg, "gain", None)
    alpha = getattr(cfg, "alpha", None)
    return _Cfg(VARIANTS.index(cfg.variant), VN_MODES.index(cfg.vn_mode), int(cfg.l_max),
                1 if early_stop else 0, float(alpha) if alpha is not None else 0.0,
                float(gain.alpha_min) if gain else 0.0, float(gain.alpha_max) if gain else 0.0,
                float(gain.eta_unsat) if gain else 0.0)


def sample_errors(n, epsilon, seed, start, count):
    out = np.zeros((count, n), dtype=np.uint8)
    rc = lib().qsgo_sample_errors(n, float(epsilon), seed & (2**64 - 1), start, count, _ptr(out))
    if rc:
        raise ValueError("bad sample_errors arguments")
    return out


def philox_block(ctr, key):
    c = np.array(ctr, dtype=np.uint64)
    k = np.array(key, dtype=np.uint64)
    out = np.zeros(4, dtype=np.uint64)
    lib().qsgo_philox4x64_10(_ptr(c), _ptr(k), _ptr(out))
    return out


def syndromes_of(graph, e):
    g = _as_graph(graph)
    e = np.ascontiguousarray(e, dtype=np.uint8)
    syn = np.zeros((e.shape[0], g.m), dtype=np.uint8)
    lib().qsgo_syndromes_of(C.byref(g.c), _ptr(e), e.shape[0], _ptr(syn))
    return syn


@dataclass
class OracleResult:
    success: np.ndarray
    e_hat: np.ndarray
    iterations: np.ndarray
    unsat: np.ndarray | None = None
    vn_msgs: np.ndarray | None = None
    cn_msgs: np.ndarray | None = None
    counts: np.ndarray | None = None

    def gamma_traces(self, m):
        return [self.unsat[b, : self.counts[b, 0]] / m for b in range(len(self.success))]


def decode(graph, syndromes, l0, cfg, *, precision=32, early_stop=True, trace=False,
           capture=False, nthreads=None):
    """decode_batch (decoder.py:374-485) restated in C; precision 32 or 64."""
    g = _as_graph(graph)
    syn = np.ascontiguousarray(syndromes, dtype=np.uint8)
    if syn.ndim != 2 or syn.shape[1] != g.m:
        raise ValueError(f"syndromes must have shape (B, {g.m})")
    B = syn.shape[0]
    L = int(cfg.l_max)
    ft = np.float32 if precision == 32 else np.float64
    res = OracleResult(np.zeros(B, dtype=np.uint8), np.zeros((B, g.n), dtype=np.uint8),
                       np.zeros(B, dtype=np.int64))
    tr = None
    if trace or capture:
        res.unsat = np.zeros((B, L), dtype=np.int32)
        res.counts = np.zeros((B, 2), dtype=np.int32)
        if capture:
            res.vn_msgs = np.zeros((B, L, g.E), dtype=ft)
            res.cn_msgs = np.zeros((B, L, g.E), dtype=ft)
        tr = _Trace(_ptr(res.unsat), _ptr(res.vn_msgs), _ptr(res.cn_msgs), _ptr(res.counts))
    c = _cfg(cfg, early_stop)
    nt = nthreads or min(os.cpu_count() or 1, max(1, B // 64))
    fn = lib().qsgo32_decode if precision == 32 else lib().qsgo64_decode
    rc = fn(C.byref(g.c), C.byref(c), float(l0), _ptr(syn), B, _ptr(res.success),
            _ptr(res.e_hat), _ptr(res.iterations), C.byref(tr) if tr else None, nt)
    if rc:
        raise RuntimeError(f"oracle decode failed rc={rc}")
    res.success = res.success.astype(bool)
    return res


def frames(graph, cfg, epsilon, epsilon0, seed, start, count, *, precision=32,
           want_ehat=False, nthreads=None):
    """harness._decode_frames restated; returns (fails, iters, e_hat, counters)."""
    g = _as_graph(graph)
    fails = np.zeros(count, dtype=np.uint8)
    iters = np.zeros(count, dtype=np.int64)
    ehat = np.zeros((count, g.n), dtype=np.uint8) if want_ehat else None
    counters = np.zeros(4, dtype=np.int64)
    c = _cfg(cfg, True)
    nt = nthreads or (os.cpu_count() or 1)
    fn = lib().qsgo32_frames if precision == 32 else lib().qsgo64_frames
    rc = fn(C.byref(g.c), C.byref(c), float(epsilon), float(epsilon0), seed & (2**64 - 1),
            start, count, _ptr(fails), _ptr(iters), _ptr(ehat), _ptr(counters), nt)
    if rc:
        raise RuntimeError(f"oracle frames failed rc={rc}")
    return fails.astype(bool), iters, ehat, counters


def prior_llr(epsilon0):
    """channel.py:48-52."""
    return math.log(3.0 * (1.0 - epsilon0) / epsilon0)


MATH_FUNCS = {"exp_neg": 0, "log1p_01": 1, "log1p": 2, "expm1": 3, "logaddexp": 4, "vnF": 6}


def math32(name, x, y=None):
    x = np.ascontiguousarray(x, dtype=np.float32)
    y = np.ascontiguousarray(y if y is not None else x, dtype=np.float32)
    out = np.empty_like(x)
    lib().qsgo_math32_batch(MATH_FUNCS[name], _ptr(x), _ptr(y), _ptr(out), x.size)
    return out


def bp4_mags(x):
    """Output magnitudes of one BP4 check for input magnitudes x (the fp32
    product-form recipe, qo_bp4_mags)."""
    x = np.ascontiguousarray(x, dtype=np.float32)
    out = np.empty_like(x)
    lib().qsgo_bp4_mags(_ptr(x), x.size, _ptr(out))
    return out
