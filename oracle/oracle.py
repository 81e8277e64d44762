"""ctypes front-end of the C restatement (oracle/vlq_oracle.c) -- TEST INFRASTRUCTURE.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may use
this module; it is the parity checker, never the thing measured or shipped.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

from . import vlq1

HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = None


class _VoIndex(ctypes.Structure):
    _fields_ = [
        ("dim", ctypes.c_uint32), ("k", ctypes.c_uint32), ("n", ctypes.c_uint32), ("m", ctypes.c_uint32),
        ("clamp", ctypes.c_int), ("lo", ctypes.c_float), ("hi", ctypes.c_float),
        ("centroids", ctypes.c_void_p), ("nbr", ctypes.c_void_p), ("elen", ctypes.c_void_p),
        ("pq", ctypes.c_void_p), ("t2", ctypes.c_void_p), ("t3", ctypes.c_void_p),
        ("list_off", ctypes.c_void_p), ("ids", ctypes.c_void_p), ("codes", ctypes.c_void_p),
        ("lambdas", ctypes.c_void_p),
    ]


def lib():
    global _LIB
    if _LIB is None:
        path = os.path.join(HERE, "liboracle.so")
        if not os.path.exists(path):
            raise RuntimeError(f"oracle not built: {path} (run make -C oracle)")
        L = ctypes.CDLL(path)
        L.vo_last_error.restype = ctypes.c_char_p
        L.vo_quantize_lambda.restype = ctypes.c_uint8
        L.vo_quantize_lambda.argtypes = [ctypes.c_float, ctypes.c_float, ctypes.c_float]
        L.vo_dequantize_lambda.restype = ctypes.c_float
        L.vo_dequantize_lambda.argtypes = [ctypes.c_uint8, ctypes.c_float, ctypes.c_float]
        L.vo_w2.restype = ctypes.c_uint32
        L.vo_w2.argtypes = [ctypes.c_uint32, ctypes.c_float, ctypes.c_uint32]
        L.vo_line_lambda_raw.restype = ctypes.c_float
        L.vo_line_lambda_raw.argtypes = [ctypes.c_float] * 3
        L.vo_line_sqdist_raw.restype = ctypes.c_float
        L.vo_line_sqdist_raw.argtypes = [ctypes.c_float] * 4
        L.vo_direct_adc.restype = ctypes.c_float
        L.vo_direct_adc.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_uint8,
                                    ctypes.c_uint32, ctypes.c_uint32]
        L.vo_adc_distance.restype = ctypes.c_float
        L.vo_adc_distance.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                      ctypes.c_uint8, ctypes.c_uint32, ctypes.c_uint32]
        _LIB = L
    return _LIB


def _p(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p) if a is not None else None


def _check(rc: int):
    if rc != 0:
        raise RuntimeError(lib().vo_last_error().decode())


def compute_t2(pq: np.ndarray) -> np.ndarray:
    m, ksub, dsub = pq.shape
    t2 = np.empty((m, ksub), np.float32)
    _check(lib().vo_compute_t2(_p(np.ascontiguousarray(pq, np.float32)), ctypes.c_uint32(m * dsub),
                               ctypes.c_uint32(m), _p(t2)))
    return t2


def compute_t3(centroids: np.ndarray, pq: np.ndarray) -> np.ndarray:
    k, dim = centroids.shape
    m = pq.shape[0]
    t3 = np.empty((k, m, vlq1.KSUB), np.float32)
    _check(lib().vo_compute_t3(_p(np.ascontiguousarray(centroids, np.float32)), ctypes.c_uint32(k),
                               ctypes.c_uint32(dim), _p(np.ascontiguousarray(pq, np.float32)),
                               ctypes.c_uint32(m), _p(t3)))
    return t3


class OracleIndex:
    """A VLQ1 index held in the flat SoA layout, searched by the C oracle."""

    def __init__(self, ix: vlq1.Vlq1):
        self.ix = ix
        self.t2 = compute_t2(ix.pq)
        self.t3 = ix.t3 if ix.t3 is not None else compute_t3(ix.centroids, ix.pq)
        if ix.list_off is None:
            ix.list_off = np.zeros(ix.k * ix.n + 1, np.uint64)
            ix.ids = np.zeros(0, np.uint32)
            ix.codes = np.zeros((0, ix.m), np.uint8)
            ix.lambdas = np.zeros(0, np.uint8)
        self._keep = [np.ascontiguousarray(a) for a in (ix.centroids, ix.nbr, ix.elen, ix.pq, self.t2,
                                                        self.t3, ix.list_off, ix.ids, ix.codes, ix.lambdas)]
        c = self._keep
        self.s = _VoIndex(ix.dim, ix.k, ix.n, ix.m, int(ix.clamp), ix.lo, ix.hi, *[_p(a) for a in c])

    @classmethod
    def load(cls, path: str) -> "OracleIndex":
        return cls(vlq1.read(path))

    def search(self, queries: np.ndarray, w1: int = 64, alpha: float = 0.25, k: int = 10,
               threads: int = 0):
        q = np.ascontiguousarray(queries, np.float32)
        if q.ndim != 2:
            raise RuntimeError("expected a 2-D float array")
        if q.shape[1] != self.ix.dim:
            raise RuntimeError("search_batch: dimension mismatch")
        nq = q.shape[0]
        ids = np.empty((nq, k), np.int64)
        dists = np.empty((nq, k), np.float32)
        scanned = np.zeros(nq, np.uint64)
        _check(lib().vo_search(ctypes.byref(self.s), _p(q), ctypes.c_uint64(nq), ctypes.c_uint32(w1),
                               ctypes.c_float(alpha), ctypes.c_uint32(k), _p(ids), _p(dists), _p(scanned),
                               ctypes.c_int(threads)))
        return ids, dists, scanned

    def first_level(self, queries: np.ndarray, w1: int, threads: int = 0) -> np.ndarray:
        """Exact top-w1 region ids of every query (first_level_scan,
        search.cpp:11-36), uint32 [nq, w1] in (dist, id) order."""
        q = np.ascontiguousarray(queries, np.float32)
        top = np.empty((q.shape[0], w1), np.uint32)
        _check(lib().vo_first_level(ctypes.byref(self.s), _p(q), ctypes.c_uint64(q.shape[0]), ctypes.c_uint32(w1),
                                    _p(top), ctypes.c_int(threads)))
        return top

    def search_from_top(self, queries: np.ndarray, top: np.ndarray, w1: int, alpha: float, k: int,
                        threads: int = 0):
        """search() from given top-w1 lists (search.cpp:38-167)."""
        q = np.ascontiguousarray(queries, np.float32)
        top = np.ascontiguousarray(top, np.uint32)
        assert top.shape == (q.shape[0], w1)
        nq = q.shape[0]
        ids = np.empty((nq, k), np.int64)
        dists = np.empty((nq, k), np.float32)
        scanned = np.zeros(nq, np.uint64)
        _check(lib().vo_search_from_top(ctypes.byref(self.s), _p(q), ctypes.c_uint64(nq), ctypes.c_uint32(w1),
                                        ctypes.c_float(alpha), ctypes.c_uint32(k), _p(top), _p(ids), _p(dists),
                                        _p(scanned), ctypes.c_int(threads)))
        return ids, dists, scanned

    def select(self, queries: np.ndarray, w1: int, alpha: float, threads: int = 0):
        """first_level_scan + second_level_rank: (sel uint32 [nq, w2], ab
        float32 [nq, w2, 2]) -- the select-split hand-off."""
        q = np.ascontiguousarray(queries, np.float32)
        w2 = int(lib().vo_w2(w1, np.float32(alpha), self.ix.n))
        sel = np.empty((q.shape[0], w2), np.uint32)
        ab = np.empty((q.shape[0], w2, 2), np.float32)
        _check(lib().vo_select(ctypes.byref(self.s), _p(q), ctypes.c_uint64(q.shape[0]), ctypes.c_uint32(w1),
                               ctypes.c_float(alpha), _p(sel), _p(ab), ctypes.c_int(threads)))
        return sel, ab

    def search_from_sel(self, queries: np.ndarray, sel: np.ndarray, ab: np.ndarray, w1: int, alpha: float, k: int,
                        threads: int = 0):
        """query_term5 .. select_topk from a select() hand-off (on this index's lists)."""
        q = np.ascontiguousarray(queries, np.float32)
        nq = q.shape[0]
        sel = np.ascontiguousarray(sel, np.uint32)
        ab = np.ascontiguousarray(ab, np.float32)
        ids = np.empty((nq, k), np.int64)
        d = np.empty((nq, k), np.float32)
        sc = np.empty(nq, np.uint64)
        _check(lib().vo_search_from_sel(ctypes.byref(self.s), _p(q), ctypes.c_uint64(nq), ctypes.c_uint32(w1),
                                        ctypes.c_float(alpha), ctypes.c_uint32(k), _p(sel), _p(ab), _p(ids), _p(d),
                                        _p(sc), ctypes.c_int(threads)))
        return ids, d, sc

    def ivf_build(self, base: np.ndarray):
        """build_ivf_baseline (ivf_baseline.cpp:11-51) with this model's
        codebook and PQ -> (list_off u64[k+1], ids u32[N], codes u8[N, m])."""
        x = np.ascontiguousarray(base, np.float32)
        nb = x.shape[0]
        off = np.zeros(self.ix.k + 1, np.uint64)
        ids = np.empty(nb, np.uint32)
        codes = np.empty((nb, self.ix.m), np.uint8)
        _check(lib().vo_ivf_build(ctypes.byref(self.s), _p(x), ctypes.c_uint64(nb), _p(off), _p(ids), _p(codes)))
        return off, ids, codes

    def ivf_search(self, lists, queries: np.ndarray, w: int, k: int, threads: int = 0):
        """search_ivf_baseline (ivf_baseline.cpp:53-126) over `lists` (from
        ivf_build) -> (ids int64[nq,k], dists float32[nq,k], scanned u64[nq])."""
        off, ids_, codes = (np.ascontiguousarray(a) for a in lists)
        q = np.ascontiguousarray(queries, np.float32)
        nq = q.shape[0]
        ids = np.empty((nq, k), np.int64)
        dists = np.empty((nq, k), np.float32)
        scanned = np.zeros(nq, np.uint64)
        _check(lib().vo_ivf_search(ctypes.byref(self.s), _p(off), _p(ids_), _p(codes), _p(q), ctypes.c_uint64(nq),
                                   ctypes.c_uint32(w), ctypes.c_uint32(k), _p(ids), _p(dists), _p(scanned),
                                   ctypes.c_int(threads)))
        return ids, dists, scanned

    def assign(self, base: np.ndarray, clamp: bool | None = None, threads: int = 0):
        """Per-point (cell, exact lambda, code, lambda byte) of the add path."""
        x = np.ascontiguousarray(base, np.float32)
        nb = x.shape[0]
        cells = np.empty(nb, np.uint32)
        lams = np.empty(nb, np.float32)
        codes = np.empty((nb, self.ix.m), np.uint8)
        lb = np.empty(nb, np.uint8)
        cl = self.ix.clamp if clamp is None else clamp
        _check(lib().vo_assign(ctypes.byref(self.s), _p(x), ctypes.c_uint64(nb), ctypes.c_int(int(cl)),
                               _p(cells), _p(lams), _p(codes), _p(lb), ctypes.c_int(threads)))
        return cells, lams, codes, lb

    def observe_lambda_range(self, base: np.ndarray, threads: int = 0):
        """observe_lambda_range (index.cpp:110-132)."""
        x = np.ascontiguousarray(base, np.float32)
        nb = x.shape[0]
        if nb == 0:
            return 0.0, 1.0
        cells = np.empty(nb, np.uint32)
        lams = np.empty(nb, np.float32)
        _check(lib().vo_assign(ctypes.byref(self.s), _p(x), ctypes.c_uint64(nb), ctypes.c_int(0), _p(cells),
                               _p(lams), None, None, ctypes.c_int(threads)))
        lo, hi = np.float32(lams.min()), np.float32(lams.max())
        if not lo < hi:
            return float(lo), float(np.float32(lo + np.float32(1.0)))
        return float(lo), float(hi)

    def build(self, base: np.ndarray, threads: int = 0) -> vlq1.Vlq1:
        """build_index (index.cpp:134-203) on this model: lists ordered by point id."""
        ix = self.ix
        lo, hi = (ix.lo, ix.hi)
        model = self
        if not ix.clamp:
            lo, hi = self.observe_lambda_range(base, threads)
            model = OracleIndex(vlq1.Vlq1(ix.dim, ix.k, ix.n, ix.m, ix.clamp, lo, hi, ix.centroids, ix.nbr,
                                          ix.elen, ix.pq, self.t3))
        cells, _, codes, lb = model.assign(base, threads=threads)
        order = np.argsort(cells, kind="stable")
        counts = np.bincount(cells, minlength=ix.k * ix.n).astype(np.uint64)
        off = np.zeros(ix.k * ix.n + 1, np.uint64)
        np.cumsum(counts, out=off[1:])
        return vlq1.Vlq1(ix.dim, ix.k, ix.n, ix.m, ix.clamp, lo, hi, ix.centroids, ix.nbr, ix.elen, ix.pq,
                         None, off, order.astype(np.uint32), codes[order], lb[order])

    def query_tables(self, y: np.ndarray):
        y = np.ascontiguousarray(y, np.float32)
        ws = np.empty(self.ix.k, np.float32)
        t5 = np.empty((self.ix.m, vlq1.KSUB), np.float32)
        lib().vo_query_tables(ctypes.byref(self.s), _p(y), _p(ws), _p(t5))
        return ws, t5

    def adc_distance(self, ws, t5, code, lambda_byte, i, j) -> float:
        code = np.ascontiguousarray(code, np.uint8)
        return float(lib().vo_adc_distance(ctypes.byref(self.s), _p(ws), _p(t5), _p(code), lambda_byte, i, j))

    def direct_adc(self, y, code, lambda_byte, i, j) -> float:
        y = np.ascontiguousarray(y, np.float32)
        code = np.ascontiguousarray(code, np.uint8)
        return float(lib().vo_direct_adc(ctypes.byref(self.s), _p(y), _p(code), lambda_byte, i, j))


def quantize_lambda(lam: float, lo: float, hi: float) -> int:
    return int(lib().vo_quantize_lambda(lam, lo, hi))


def dequantize_lambda(b: int, lo: float, hi: float) -> float:
    return float(lib().vo_dequantize_lambda(b, lo, hi))


def w2(w1: int, alpha: float, n: int) -> int:
    return int(lib().vo_w2(w1, alpha, n))


def line_lambda(a: float, b: float, c: float) -> float:
    return float(lib().vo_line_lambda_raw(a, b, c))


def line_sqdist(a: float, b: float, c: float, lam: float) -> float:
    return float(lib().vo_line_sqdist_raw(a, b, c, lam))


# ---- k-means restatement (oracle/train_oracle.cpp, kmeans.cpp) ---------------
_TLIB = None


def train_lib():
    global _TLIB
    if _TLIB is None:
        path = os.path.join(HERE, "liboracle_train.so")
        if not os.path.exists(path):
            raise RuntimeError(f"oracle not built: {path} (run make -C oracle)")
        L = ctypes.CDLL(path)
        L.vo_train_last_error.restype = ctypes.c_char_p
        for f in ("vo_train_kmeans", "vo_kmeans_seed", "vo_kmeans_lloyd"):
            getattr(L, f).restype = ctypes.c_int
        L.vo_train_kmeans.argtypes = [ctypes.c_void_p, ctypes.c_uint64, ctypes.c_uint32, ctypes.c_uint32,
                                      ctypes.c_uint32, ctypes.c_uint64, ctypes.c_void_p]
        L.vo_kmeans_seed.argtypes = [ctypes.c_void_p, ctypes.c_uint64, ctypes.c_uint32, ctypes.c_uint32,
                                     ctypes.c_uint64, ctypes.c_void_p]
        L.vo_kmeans_lloyd.argtypes = [ctypes.c_void_p, ctypes.c_uint64, ctypes.c_uint32, ctypes.c_uint32,
                                      ctypes.c_uint32, ctypes.c_void_p, ctypes.c_void_p]
        L.vo_quantization_error.restype = ctypes.c_double
        L.vo_quantization_error.argtypes = [ctypes.c_void_p, ctypes.c_uint64, ctypes.c_uint32, ctypes.c_void_p,
                                            ctypes.c_uint32]
        _TLIB = L
    return _TLIB


def _tcheck(rc: int):
    if rc != 0:
        raise RuntimeError(train_lib().vo_train_last_error().decode())


def train_kmeans(x: np.ndarray, k: int, iters: int, seed: int) -> np.ndarray:
    """train_kmeans (kmeans.cpp:104-185), the reference's random stream included."""
    x = np.ascontiguousarray(x, np.float32)
    out = np.empty((k, x.shape[1]), np.float32)
    _tcheck(train_lib().vo_train_kmeans(_p(x), x.shape[0], x.shape[1], k, iters, seed, _p(out)))
    return out


def kmeans_seed(x: np.ndarray, k: int, seed: int) -> np.ndarray:
    """seed_centroids (kmeans.cpp:54-102): the reference's k-means++ seeds."""
    x = np.ascontiguousarray(x, np.float32)
    out = np.empty((k, x.shape[1]), np.float32)
    _tcheck(train_lib().vo_kmeans_seed(_p(x), x.shape[0], x.shape[1], k, seed, _p(out)))
    return out


def kmeans_lloyd(x: np.ndarray, init: np.ndarray, iters: int) -> np.ndarray:
    """The Lloyd + empty-cluster repair loop (kmeans.cpp:117-183) from init."""
    x = np.ascontiguousarray(x, np.float32)
    init = np.ascontiguousarray(init, np.float32)
    out = np.empty_like(init)
    _tcheck(train_lib().vo_kmeans_lloyd(_p(x), x.shape[0], x.shape[1], init.shape[0], iters, _p(init), _p(out)))
    return out


def quantization_error(x: np.ndarray, centroids: np.ndarray) -> float:
    """quantization_error (kmeans.cpp:35-51)."""
    x = np.ascontiguousarray(x, np.float32)
    c = np.ascontiguousarray(centroids, np.float32)
    return float(train_lib().vo_quantization_error(_p(x), x.shape[0], x.shape[1], _p(c), c.shape[0]))
