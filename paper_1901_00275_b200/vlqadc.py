"""Drop-in ``vlqadc`` module backed by the B200 engine.

Mirrors the reference Python surface (/root/reference/proj/python/bindings.cpp
:143-233, re-exported by python/vlqadc/__init__.py:8-24):

    Index.train / Index.load / index.add / index.search / index.save
    index.k, .n, .m, .dim, .ntotal
    gen_synthetic, brute_force_gt, read_vecs, write_vecs, set_max_threads

Argument names, defaults, return shapes/dtypes, padding (-1 / +inf) and the
error texts (raised as RuntimeError) follow the reference.  Everything that
computes runs in libvlqgpu.so on the GPU; there is no CPU fallback.

Extensions beyond the reference API (for sharding, benchmarks and parity
tests) are keyword-only or separately named: ``Index.from_model``,
``Index.search_device``, ``Index.encode``, ``Index.lists``,
``shard_rank/shard_count`` and ``device`` on the constructors.
"""
from __future__ import annotations

import ctypes
import os
import struct

import numpy as np

from . import _lib

KSUB = 256


def _default_device() -> int:
    for var in ("VLQ_DEVICE", "LOCAL_RANK"):
        if var in os.environ:
            return int(os.environ[var])
    return 0


def _p(a: np.ndarray | None):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


CUDA_STREAM_LEGACY = 0x1  # cudaStreamLegacy: the legacy default stream (torch's default stream)


def _stream(stream: int | None):
    """None -> the engine's own stream; 0 (torch's default stream handle) ->
    cudaStreamLegacy, so work stays ordered with torch's default stream;
    anything else -> that cudaStream_t."""
    if stream is None:
        return None
    return ctypes.c_void_p(CUDA_STREAM_LEGACY if stream == 0 else stream)


def _to_vecset(arr, validate: bool = True) -> np.ndarray:
    """to_vecset + VectorSet::validate (bindings.cpp:23-31, vecset.cpp:8-20).
    validate=False leaves the finiteness check to the engine (the host search
    checks while staging the queries, with the same message)."""
    a = np.ascontiguousarray(arr, dtype=np.float32)
    if a.ndim != 2:
        raise RuntimeError("expected a 2-D float array")
    if validate and a.size and not np.isfinite(a).all():
        raise RuntimeError("VectorSet: non-finite value")
    return a


class Index:
    """Two-level (vector + line quantization) inverted index on one B200."""

    def __init__(self, *, device: int | None = None, shard_rank: int = 0, shard_count: int = 1,
                 workspace_bytes: int = 0, max_tile: int = 0, force_exact: bool = False):
        L = _lib.lib()
        cfg = _lib.VlqConfig(_default_device() if device is None else device, shard_rank, shard_count,
                             workspace_bytes, max_tile, int(force_exact))
        h = ctypes.c_void_p()
        _lib.check(L.vlq_engine_create(ctypes.byref(cfg), ctypes.byref(h)))
        self._h = h
        self._device = cfg.device

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            try:
                _lib.lib().vlq_engine_destroy(h)
            except Exception:
                pass
            self._h = None

    # ---- construction -------------------------------------------------------
    @staticmethod
    def train(train, k: int = 1024, n: int = 16, m: int = 8, iters: int = 10, seed: int = 42,
              clamp_lambda: bool = True, **engine_kw) -> "Index":
        """Index.train (bindings.cpp:44-81), on the GPU (csrc/train.cu).  Same
        pipeline (k-means++ seeding, Lloyd, empty-cluster repair, n-NN graph,
        PQ) and error texts as the reference; the codebooks equal the
        reference's in distribution, not bit for bit (the seeding's random
        stream differs)."""
        t = _to_vecset(train)
        if m == 0 or t.shape[1] % m != 0:
            raise RuntimeError("m must divide the vector dimension")
        idx = Index(**engine_kw)
        _lib.check(_lib.lib().vlq_engine_train(idx._h, _p(t), t.shape[0], t.shape[1], k, n, m, iters, seed,
                                               int(clamp_lambda)))
        return idx

    @staticmethod
    def load(path: str, **engine_kw) -> "Index":
        """Index.load: VLQ1 deserialize_index (index_io.cpp:100-159)."""
        idx = Index(**engine_kw)
        _lib.check(_lib.lib().vlq_engine_load_vlq1(idx._h, os.fsencode(str(path))))
        return idx

    @staticmethod
    def from_model(dim: int, k: int, n: int, m: int, clamp: bool, lo: float, hi: float, centroids, nbr, elen, pq,
                   t3=None, **engine_kw) -> "Index":
        """An empty index over trained quantizers (a VLQ1 'model')."""
        idx = Index(**engine_kw)
        cent = np.ascontiguousarray(centroids, np.float32)
        nb = np.ascontiguousarray(nbr, np.uint32)
        el = np.ascontiguousarray(elen, np.float32)
        pqa = np.ascontiguousarray(pq, np.float32)
        t3a = None if t3 is None else np.ascontiguousarray(t3, np.float32)
        _lib.check(_lib.lib().vlq_engine_set_model(idx._h, dim, k, n, m, int(clamp), lo, hi, _p(cent), _p(nb),
                                                   _p(el), _p(pqa), _p(t3a)))
        return idx

    # ---- the reference API --------------------------------------------------
    def add(self, base) -> None:
        """Index.add (bindings.cpp:83-97): ids are the row numbers."""
        b = _to_vecset(base)
        _lib.check(_lib.lib().vlq_engine_add(self._h, _p(b), b.shape[0], b.shape[1]))

    def add_vecs(self, path: str, chunk_rows: int = 0) -> None:
        """add(read_vecs(path)) streamed from the file (.fvecs / .bvecs /
        .ivecs) without holding the base in host memory (extension)."""
        _lib.check(_lib.lib().vlq_engine_add_vecs(self._h, str(path).encode(), chunk_rows))

    def search(self, queries, w1: int = 64, alpha: float = 0.25, k: int = 10, *, return_scanned: bool = False):
        """Index.search (bindings.cpp:99-126) -> (ids int64[nq,k], dists float32[nq,k])."""
        q = _to_vecset(queries, validate=False)  # vlq_engine_search validates while staging
        nq = q.shape[0]
        ids = np.empty((nq, k), np.int64)
        dists = np.empty((nq, k), np.float32)
        scanned = np.zeros(nq, np.uint64)
        dim = q.shape[1] if q.size else self.dim
        if q.shape[1] != self.dim:
            _to_vecset(q)  # the reference validates (non-finite) before the dimension check
            raise RuntimeError("search_batch: dimension mismatch")
        _lib.check(_lib.lib().vlq_engine_search(self._h, _p(q), nq, dim, w1, alpha, k, _p(ids), _p(dists),
                                                _p(scanned)))
        if return_scanned:
            return ids, dists, scanned
        return ids, dists

    def save(self, path: str) -> None:
        """Index.save: serialize_index with t3 stored (bindings.cpp:128-131)."""
        _lib.check(_lib.lib().vlq_engine_save_vlq1(self._h, os.fsencode(str(path)), 1))

    def _info(self) -> _lib.VlqInfo:
        info = _lib.VlqInfo()
        _lib.check(_lib.lib().vlq_engine_info(self._h, ctypes.byref(info)))
        return info

    @property
    def k(self) -> int:
        return int(self._info().k)

    @property
    def n(self) -> int:
        return int(self._info().n)

    @property
    def m(self) -> int:
        return int(self._info().m)

    @property
    def dim(self) -> int:
        return int(self._info().dim)

    @property
    def ntotal(self) -> int:
        return int(self._info().ntotal)

    # ---- extensions ------------------------------------------------------------
    @property
    def device(self) -> int:
        return self._device

    @property
    def lambda_range(self) -> tuple[float, float]:
        info = self._info()
        return float(info.lambda_lo), float(info.lambda_hi)

    @property
    def local_entries(self) -> int:
        return int(self._info().local_entries)

    def search_device(self, d_queries: int, nq: int, w1: int, alpha: float, k: int, d_ids: int, d_dists: int,
                      d_scanned: int | None = None, stream: int | None = None) -> None:
        """Asynchronous search on device pointers (e.g. torch tensors' data_ptr())."""
        _lib.check(_lib.lib().vlq_engine_search_device(self._h, ctypes.c_void_p(d_queries), nq, w1, alpha, k,
                                                       ctypes.c_void_p(d_ids), ctypes.c_void_p(d_dists),
                                                       ctypes.c_void_p(d_scanned) if d_scanned else None,
                                                       _stream(stream)))

    def search_coarse_device(self, d_queries: int, nq: int, w1: int, d_top: int, stream: int | None = None) -> None:
        """first_level_scan only (search.cpp:11-36): exact top-w1 region ids
        (uint32 [nq, w1], (dist, id) order) into d_top.  Asynchronous."""
        _lib.check(_lib.lib().vlq_engine_search_coarse_device(self._h, ctypes.c_void_p(d_queries), nq, w1,
                                                              ctypes.c_void_p(d_top),
                                                              _stream(stream)))

    def search_fine_device(self, d_queries: int, nq: int, w1: int, alpha: float, k: int, d_top: int, d_ids: int,
                           d_dists: int, d_scanned: int | None = None, stream: int | None = None) -> None:
        """The rest of the search (search.cpp:38-167) on this shard from given
        top-w1 lists.  search_coarse_device + search_fine_device ==
        search_device.  Asynchronous."""
        _lib.check(_lib.lib().vlq_engine_search_fine_device(self._h, ctypes.c_void_p(d_queries), nq, w1, alpha, k,
                                                            ctypes.c_void_p(d_top), ctypes.c_void_p(d_ids),
                                                            ctypes.c_void_p(d_dists),
                                                            ctypes.c_void_p(d_scanned) if d_scanned else None,
                                                            _stream(stream)))

    def search_select_device(self, d_queries: int, nq: int, w1: int, alpha: float, d_sel: int, d_ab: int,
                             stream: int | None = None) -> None:
        """first_level_scan + second_level_rank (search.cpp:11-78): the selected
        cells (uint32 [nq, w2]) and their exact (a, b) distances (float32
        [nq, w2, 2]) into d_sel / d_ab.  Asynchronous."""
        _lib.check(_lib.lib().vlq_engine_search_select_device(self._h, ctypes.c_void_p(d_queries), nq, w1, alpha,
                                                              ctypes.c_void_p(d_sel), ctypes.c_void_p(d_ab),
                                                              _stream(stream)))

    def search_fine_sel_device(self, d_queries: int, nq: int, w1: int, alpha: float, k: int, d_sel: int, d_ab: int,
                               d_ids: int, d_dists: int, d_scanned: int | None = None,
                               stream: int | None = None) -> None:
        """query_term5 .. select_topk (search.cpp:80-167) on this shard from a
        given selection.  search_select_device + search_fine_sel_device ==
        search_device.  Asynchronous."""
        _lib.check(_lib.lib().vlq_engine_search_fine_sel_device(self._h, ctypes.c_void_p(d_queries), nq, w1, alpha,
                                                                k, ctypes.c_void_p(d_sel), ctypes.c_void_p(d_ab),
                                                                ctypes.c_void_p(d_ids), ctypes.c_void_p(d_dists),
                                                                ctypes.c_void_p(d_scanned) if d_scanned else None,
                                                                _stream(stream)))

    def w2(self, w1: int, alpha: float) -> int:
        """Cells scanned per query (QueryParams::w2, search.hpp:16-20)."""
        return int(_lib.lib().vlq_w2(w1, alpha, self.n))

    def set_tuning(self, key: str, value: int) -> None:
        """Study knobs (scan_variant, scan_slots, tc_search_min_k, force_exact);
        results are identical for every setting."""
        _lib.check(_lib.lib().vlq_engine_set_tuning(self._h, key.encode(), int(value)))

    def sync(self, stream: int | None = None) -> None:
        _lib.check(_lib.lib().vlq_engine_sync(self._h, _stream(stream)))

    def add_synthetic(self, n: int, clusters: int = 200, spread: float = 0.05, seed: int = 42) -> None:
        """Streamed add of n rows of the device synthetic generator."""
        _lib.check(_lib.lib().vlq_engine_add_synthetic(self._h, n, clusters, spread, seed))

    def set_profiling(self, on: bool = True) -> None:
        _lib.check(_lib.lib().vlq_engine_set_profiling(self._h, int(on)))

    def stats(self, reset: bool = False) -> dict:
        s = _lib.VlqStats()
        _lib.check(_lib.lib().vlq_engine_get_stats(self._h, ctypes.byref(s)))
        if reset:
            _lib.check(_lib.lib().vlq_engine_reset_stats(self._h))
        return {"launches": int(s.launches), "tiles": int(s.tiles), "flagged": int(s.flagged),
                "tc_fallbacks": int(s.tc_fallbacks),
                "phase_ms": dict(zip(_lib.PHASES, [float(x) for x in s.phase_ms]))}

    def encode(self, x):
        """Per-point (cell, exact lambda, code, lambda byte) of the add path."""
        a = _to_vecset(x)
        nx = a.shape[0]
        m = self.m
        cells = np.empty(nx, np.uint32)
        lams = np.empty(nx, np.float32)
        codes = np.empty((nx, m), np.uint8)
        lb = np.empty(nx, np.uint8)
        _lib.check(_lib.lib().vlq_engine_encode(self._h, _p(a), nx, _p(cells), _p(lams), _p(codes), _p(lb)))
        return cells, lams, codes, lb

    def model(self) -> dict:
        """The trained quantizers (host copies): centroids, nbr, elen, pq, lambda range, clamp."""
        info = self._info()
        k, n, m, dim = int(info.k), int(info.n), int(info.m), int(info.dim)
        cent = np.empty((k, dim), np.float32)
        nbr = np.empty((k, n), np.uint32)
        elen = np.empty((k, n), np.float32)
        pq = np.empty((m, KSUB, dim // m), np.float32)
        _lib.check(_lib.lib().vlq_engine_get_model(self._h, _p(cent), _p(nbr), _p(elen), _p(pq)))
        return dict(dim=dim, k=k, n=n, m=m, clamp=bool(info.clamp_lambda), lo=float(info.lambda_lo),
                    hi=float(info.lambda_hi), centroids=cent, nbr=nbr, elen=elen, pq=pq)

    def list_offsets(self) -> np.ndarray:
        """This engine's list offsets u64[k*n+1] only (cell c holds entries
        [off[c], off[c+1]))."""
        info = self._info()
        off = np.empty(info.k * info.n + 1, np.uint64)
        _lib.check(_lib.lib().vlq_engine_get_lists(self._h, _p(off), None, None, None))
        return off

    def lists(self):
        """This engine's posting lists: (list_off u64[k*n+1], ids u32, codes u8[.,m], lambdas u8)."""
        info = self._info()
        ne = int(info.local_entries)
        off = np.empty(info.k * info.n + 1, np.uint64)
        ids = np.empty(ne, np.uint32)
        codes = np.empty((ne, info.m), np.uint8)
        lams = np.empty(ne, np.uint8)
        _lib.check(_lib.lib().vlq_engine_get_lists(self._h, _p(off), _p(ids), _p(codes), _p(lams)))
        return off, ids, codes, lams


    def cells(self, cells):
        """The posting lists of the given cells, concatenated in request order:
        (counts u64[len(cells)], ids u32, codes u8[., m], lambdas u8)."""
        c = np.ascontiguousarray(cells, np.uint32).ravel()
        counts = np.empty(c.shape[0], np.uint64)
        _lib.check(_lib.lib().vlq_engine_get_cells(self._h, _p(c), c.shape[0], _p(counts), None, None, None))
        tot = int(counts.sum())
        ids = np.empty(tot, np.uint32)
        codes = np.empty((tot, self.m), np.uint8)
        lams = np.empty(tot, np.uint8)
        if tot:
            _lib.check(_lib.lib().vlq_engine_get_cells(self._h, _p(c), c.shape[0], _p(counts), _p(ids), _p(codes),
                                                       _p(lams)))
        return counts, ids, codes, lams

# ---- module functions ---------------------------------------------------------
_MAX_THREADS = 0


class IndexGroup:
    """The index sharded over several GPUs of one box, driven by ONE process
    (include/vlq_gpu.h vlq_group_*; csrc/group.cu): engine g on devices[g]
    holds the posting lists c with shard_of_cell(c, G) == g, the coarse
    quantizer is replicated; search runs the query-split selection, the
    sharded scan reading the selections over NVLink peer memory, and the
    per-slice (dist, id) merge of the shards' top-k from peer memory.
    Results equal Index.search on the unsharded index bit for bit."""

    def __init__(self, devices, *, shards: int = 0, workspace_bytes: int = 0, max_tile: int = 0,
                 force_exact: bool = False):
        """shards S divides len(devices) = G: G / S replicas of an S-way list
        sharding (0: S = G)."""
        devs = (ctypes.c_int * len(devices))(*[int(d) for d in devices])
        cfg = _lib.VlqConfig(0, 0, 1, workspace_bytes, max_tile, int(force_exact))
        h = ctypes.c_void_p()
        _lib.check(_lib.lib().vlq_group_create(devs, len(devices), shards, ctypes.byref(cfg), ctypes.byref(h)))
        self._h = h
        self.devices = [int(d) for d in devices]
        self.shards = shards or len(devices)

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            try:
                _lib.lib().vlq_group_destroy(h)
            except Exception:
                pass
            self._h = None

    @staticmethod
    def load(path: str, devices, **kw) -> "IndexGroup":  # kw: shards, workspace_bytes, ...
        g = IndexGroup(devices, **kw)
        _lib.check(_lib.lib().vlq_group_load_vlq1(g._h, os.fsencode(str(path))))
        return g

    @staticmethod
    def from_model(model: dict, devices, **kw) -> "IndexGroup":
        """An empty group over trained quantizers (Index.model() dict)."""
        g = IndexGroup(devices, **kw)
        cent = np.ascontiguousarray(model["centroids"], np.float32)
        nb = np.ascontiguousarray(model["nbr"], np.uint32)
        el = np.ascontiguousarray(model["elen"], np.float32)
        pqa = np.ascontiguousarray(model["pq"], np.float32)
        _lib.check(_lib.lib().vlq_group_set_model(g._h, model["dim"], model["k"], model["n"], model["m"],
                                                  int(model["clamp"]), model["lo"], model["hi"], _p(cent), _p(nb),
                                                  _p(el), _p(pqa), None))
        return g

    def add(self, base) -> None:
        b = _to_vecset(base)
        _lib.check(_lib.lib().vlq_group_add(self._h, _p(b), b.shape[0], b.shape[1]))

    def add_synthetic(self, n: int, clusters: int = 200, spread: float = 0.05, seed: int = 42) -> None:
        _lib.check(_lib.lib().vlq_group_add_synthetic(self._h, n, clusters, spread, seed))

    def search(self, queries, w1: int = 64, alpha: float = 0.25, k: int = 10, *, return_scanned: bool = False):
        """Index.search over the group (same outputs)."""
        q = _to_vecset(queries)
        nq = q.shape[0]
        ids = np.empty((nq, k), np.int64)
        dists = np.empty((nq, k), np.float32)
        scanned = np.empty(nq, np.uint64) if return_scanned else None
        _lib.check(_lib.lib().vlq_group_search(self._h, _p(q), nq, q.shape[1], w1, alpha, k, _p(ids), _p(dists),
                                               _p(scanned)))
        if return_scanned:
            return ids, dists, scanned.astype(np.int64)
        return ids, dists

    def set_queries(self, queries) -> None:
        q = _to_vecset(queries)
        _lib.check(_lib.lib().vlq_group_set_queries(self._h, _p(q), q.shape[0], q.shape[1]))
        self._nq = q.shape[0]

    def search_resident(self, w1: int, alpha: float, k: int) -> float:
        """Searches the batch of set_queries(); returns its device time in ms
        (max over the devices)."""
        ms = ctypes.c_float()
        _lib.check(_lib.lib().vlq_group_search_resident(self._h, w1, alpha, k, ctypes.byref(ms)))
        self._k = k
        return float(ms.value)

    def results(self):
        nq, k = self._nq, self._k
        ids = np.empty((nq, k), np.int64)
        dists = np.empty((nq, k), np.float32)
        scanned = np.empty(nq, np.uint64)
        _lib.check(_lib.lib().vlq_group_results(self._h, _p(ids), _p(dists), _p(scanned)))
        return ids, dists, scanned.astype(np.int64)

    def set_profiling(self, on: bool = True) -> None:
        _lib.check(_lib.lib().vlq_group_set_profiling(self._h, int(on)))

    def stats(self, member: int, reset: bool = False) -> dict:
        s = _lib.VlqStats()
        _lib.check(_lib.lib().vlq_group_get_stats(self._h, member, ctypes.byref(s), int(reset)))
        return {"launches": int(s.launches), "tiles": int(s.tiles), "flagged": int(s.flagged),
                "tc_fallbacks": int(s.tc_fallbacks),
                "phase_ms": dict(zip(_lib.PHASES, [float(x) for x in s.phase_ms]))}

    def __len__(self) -> int:
        return int(_lib.lib().vlq_group_size(self._h))

    def info(self, member: int = 0) -> _lib.VlqInfo:
        out = _lib.VlqInfo()
        _lib.check(_lib.lib().vlq_group_info(self._h, member, ctypes.byref(out)))
        return out

    @property
    def ntotal(self) -> int:
        return int(self.info(0).ntotal)

    def local_entries(self) -> list[int]:
        return [int(self.info(g).local_entries) for g in range(len(self))]

    @property
    def replicas(self) -> int:
        return len(self) // self.shards


class IvfBaselineIndex:
    """The IVFADC comparison baseline (proj/include/vlq/ivf_baseline.hpp):
    k posting lists of (id, PQ code of x - c_i), built with an Index's
    codebook and PQ (as eval.cpp:182 does).  Held by that Index's engine on
    its device; build with build_ivf_baseline, query with
    search_ivf_baseline."""

    def __init__(self, index: Index):
        self.index = index

    @property
    def base_count(self) -> int:
        n = ctypes.c_uint64(0)
        _lib.check(_lib.lib().vlq_engine_ivf_get_lists(self.index._h, ctypes.byref(n), None, None, None))
        return int(n.value)

    def lists(self):
        """(list_off u64[k+1], ids u32[N], codes u8[N, m]) -- region-major,
        ids ascending within a list (the reference's ids[c] / codes[c])."""
        n = self.base_count
        off = np.empty(self.index.k + 1, np.uint64)
        ids = np.empty(n, np.uint32)
        codes = np.empty((n, self.index.m), np.uint8)
        _lib.check(_lib.lib().vlq_engine_ivf_get_lists(self.index._h, None, _p(off), _p(ids), _p(codes)))
        return off, ids, codes

    def search_device(self, d_queries: int, nq: int, w: int, k: int, d_ids: int, d_dists: int,
                      d_scanned: int | None = None, stream: int | None = None) -> None:
        _lib.check(_lib.lib().vlq_engine_ivf_search_device(self.index._h, ctypes.c_void_p(d_queries), nq, w, k,
                                                           ctypes.c_void_p(d_ids), ctypes.c_void_p(d_dists),
                                                           ctypes.c_void_p(d_scanned) if d_scanned else None,
                                                           _stream(stream)))


def build_ivf_baseline(base, index: Index) -> IvfBaselineIndex:
    """build_ivf_baseline(base, codebook, pq) (ivf_baseline.cpp:11-51) with
    index's codebook and PQ."""
    b = _to_vecset(base)
    _lib.check(_lib.lib().vlq_engine_ivf_build(index._h, _p(b), b.shape[0], b.shape[1]))
    return IvfBaselineIndex(index)


def build_ivf_baseline_synthetic(n: int, index: Index, clusters: int = 200, spread: float = 0.05,
                                 seed: int = 42) -> IvfBaselineIndex:
    """The same over rows [0, n) of the device synthetic generator."""
    _lib.check(_lib.lib().vlq_engine_ivf_build_synthetic(index._h, n, clusters, spread, seed))
    return IvfBaselineIndex(index)


def search_ivf_baseline(ivf: IvfBaselineIndex, queries, w: int, top_k: int, *, return_scanned: bool = False):
    """search_ivf_baseline(index, queries, w, top_k) (ivf_baseline.cpp:53-126)
    -> (ids int64[nq, top_k], dists float32[nq, top_k]), -1 / +inf padded."""
    q = _to_vecset(queries)
    nq = q.shape[0]
    ids = np.empty((nq, top_k), np.int64)
    dists = np.empty((nq, top_k), np.float32)
    scanned = np.zeros(nq, np.uint64)
    dim = q.shape[1] if q.size else ivf.index.dim
    _lib.check(_lib.lib().vlq_engine_ivf_search(ivf.index._h, _p(q), nq, dim, w, top_k, _p(ids), _p(dists),
                                                _p(scanned)))
    if return_scanned:
        return ids, dists, scanned
    return ids, dists


def train_kmeans(train, k: int, iters: int = 10, seed: int = 42, *, init=None,
                 device: int | None = None) -> np.ndarray:
    """train_kmeans (kmeans.cpp:104-185) on the GPU -> float32 [k, dim]:
    k-means++ seeding, Lloyd iterations, the reference's empty-cluster
    repair.  With ``init`` the seeding is skipped (the Lloyd loop then equals
    the reference's bit for bit)."""
    t = _to_vecset(train)
    out = np.empty((k, t.shape[1]), np.float32)
    ini = None
    if init is not None:
        ini = np.ascontiguousarray(init, np.float32)
        if ini.shape != (k, t.shape[1]):
            raise RuntimeError("train_kmeans: init must be [k, dim]")
    _lib.check(_lib.lib().vlq_train_kmeans(_default_device() if device is None else device, _p(t), t.shape[0],
                                           t.shape[1], k, iters, seed, _p(ini), _p(out)))
    return out


def set_max_threads(threads: int) -> None:
    """set_max_threads (parallel.cpp:13-15).  The GPU engine has no CPU worker
    pool; the value is recorded and results never depend on it."""
    global _MAX_THREADS
    _MAX_THREADS = max(0, int(threads))


def gen_synthetic(count: int, dim: int, clusters: int = 200, spread: float = 0.05, seed: int = 42) -> np.ndarray:
    """gen_synthetic (dataset.cpp:13-44); bit-identical stream."""
    out = np.empty((count, dim), np.float32)
    _lib.check(_lib.lib().vlq_gen_synthetic(count, dim, clusters, spread, seed, _p(out)))
    return out


def brute_force_gt(base, queries, k: int, *, device: int | None = None) -> np.ndarray:
    """brute_force_gt (dataset.cpp:46-92) on the GPU: exact ids, ties by id."""
    b = _to_vecset(base)
    q = _to_vecset(queries)
    if b.shape[1] != q.shape[1]:
        raise RuntimeError("brute_force_gt: dimension mismatch")
    out = np.empty((q.shape[0], k), np.uint32)
    _lib.check(_lib.lib().vlq_brute_force_gt(_default_device() if device is None else device, _p(b), b.shape[0],
                                             _p(q), q.shape[0], b.shape[1], k, _p(out)))
    return out


def gen_synthetic_device(first: int, count: int, dim: int, clusters: int, spread: float, seed: int,
                         d_out: int, *, device: int | None = None, stream: int | None = None) -> None:
    """Rows [first, first+count) of the counter-based device generator."""
    _lib.check(_lib.lib().vlq_gen_synthetic_device(_default_device() if device is None else device, first, count,
                                                   dim, clusters, spread, seed, ctypes.c_void_p(d_out),
                                                   _stream(stream)))


def brute_force_gt_synthetic(nb: int, dim: int, clusters: int, spread: float, seed: int, queries, k: int, *,
                             device: int | None = None) -> np.ndarray:
    """Exact k-NN of queries against rows [0, nb) of the device generator."""
    q = _to_vecset(queries)
    out = np.empty((q.shape[0], k), np.uint32)
    _lib.check(_lib.lib().vlq_brute_force_gt_synthetic(_default_device() if device is None else device, nb, dim,
                                                       clusters, spread, seed, _p(q), q.shape[0], k, _p(out)))
    return out


def _kind(path: str) -> str:
    if path.endswith(".bvecs"):
        return "b"
    if path.endswith(".ivecs"):
        return "i"
    return "f"


def read_vecs(path: str) -> np.ndarray:
    """read_vecs (vecs_io.cpp:29-86): byte and int payloads widen to float."""
    try:
        raw = open(path, "rb").read()
    except OSError:
        raise RuntimeError(f"read_vecs: cannot open {path}") from None
    kind = _kind(path)
    vsz = 1 if kind == "b" else 4
    rows, pos, dim = [], 0, None
    while pos < len(raw):
        if pos + 4 > len(raw):
            raise RuntimeError(f"read_vecs: truncated record header in {path}")
        (d,) = struct.unpack_from("<i", raw, pos)
        pos += 4
        if d <= 0:
            raise RuntimeError(f"read_vecs: non-positive dimension in {path}")
        if dim is None:
            dim = d
        elif d != dim:
            raise RuntimeError(f"read_vecs: mismatched record dimension in {path}")
        if pos + d * vsz > len(raw):
            raise RuntimeError(f"read_vecs: truncated record payload in {path}")
        dt = {"f": "<f4", "b": np.uint8, "i": "<i4"}[kind]
        rows.append(np.frombuffer(raw, dt, count=d, offset=pos).astype(np.float32))
        pos += d * vsz
    if not rows:
        raise RuntimeError(f"read_vecs: no records in {path}")
    out = np.stack(rows)
    if not np.isfinite(out).all():
        raise RuntimeError("VectorSet: non-finite value")
    return out


def write_vecs(array, path: str) -> None:
    """write_vecs (vecs_io.cpp:88-126)."""
    a = _to_vecset(array)
    kind = _kind(path)
    n, d = a.shape
    if kind == "b":
        if ((a < 0) | (a > 255) | (a != np.floor(a))).any():
            raise RuntimeError("write_vecs: value not representable as byte")
        payload = a.astype(np.uint8)
    elif kind == "i":
        payload = a.astype(np.int32)
    else:
        payload = a
    try:
        with open(path, "wb") as f:
            hdr = np.full((n, 1), d, "<i4").view(np.uint8)
            f.write(np.concatenate([hdr, payload.view(np.uint8).reshape(n, -1)], axis=1).tobytes())
    except OSError:
        raise RuntimeError(f"write_vecs: cannot open {path}") from None


__all__ = ["Index", "brute_force_gt", "gen_synthetic", "read_vecs", "set_max_threads", "write_vecs"]
