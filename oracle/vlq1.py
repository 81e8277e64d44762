"""VLQ1 index/model files and .fvecs in numpy -- TEST INFRASTRUCTURE (checker).

Layout follows the reference writer/reader exactly
(/root/reference/proj/src/index_io.cpp:63-98 and :100-159):

    "VLQ1" | u32 version=1 | u32 flags (bit0 clamped, bit1 t3 present)
    | u32 D, K, n, m, N | f32 lo, hi | f32 codebook[K*D] | u32 nbr[K*n]
    | f32 edge_len2[K*n] | f32 pq[m*256*(D/m)] | [f32 t3[K*m*256]]
    | K*n x { u32 L; u32 ids[L]; u8 codes[L*m]; u8 lambdas[L] }

The in-memory form is the flat SoA the GPU engine and the C oracle share:
lists are concatenated in cell order with a u64 ``list_off[K*n+1]``.
"""
from __future__ import annotations

import os
import struct
from dataclasses import dataclass, field

import numpy as np

KSUB = 256
FLAG_CLAMPED = 1
FLAG_T3 = 2


@dataclass
class Vlq1:
    dim: int
    k: int
    n: int
    m: int
    clamp: bool
    lo: float
    hi: float
    centroids: np.ndarray  # f32 [k, dim]
    nbr: np.ndarray  # u32 [k, n]
    elen: np.ndarray  # f32 [k, n]
    pq: np.ndarray  # f32 [m, 256, dsub]
    t3: np.ndarray | None = None  # f32 [k, m, 256] when stored
    list_off: np.ndarray = field(default=None)  # u64 [k*n + 1]
    ids: np.ndarray = field(default=None)  # u32 [N]
    codes: np.ndarray = field(default=None)  # u8 [N, m]
    lambdas: np.ndarray = field(default=None)  # u8 [N]

    @property
    def ntotal(self) -> int:
        return int(self.ids.shape[0]) if self.ids is not None else 0


def read(path: str) -> Vlq1:
    """deserialize_index (index_io.cpp:100-159), minus validate()."""
    with open(path, "rb") as f:
        buf = f.read()
    pos = 0

    def take(nbytes: int) -> bytes:
        nonlocal pos
        if pos + nbytes > len(buf):
            raise RuntimeError(f"deserialize_index: truncated file {path}")
        out = buf[pos : pos + nbytes]
        pos += nbytes
        return out

    if take(4) != b"VLQ1":
        raise RuntimeError(f"deserialize_index: bad magic in {path}")
    (version,) = struct.unpack("<I", take(4))
    if version != 1:
        raise RuntimeError(f"deserialize_index: unsupported version in {path}")
    flags, dim, k, n, m, count = struct.unpack("<6I", take(24))
    if dim == 0 or k == 0 or n == 0 or n >= k or m == 0 or dim % m:
        raise RuntimeError(f"deserialize_index: invalid header in {path}")
    lo, hi = struct.unpack("<2f", take(8))
    dsub = dim // m
    cent = np.frombuffer(take(4 * k * dim), "<f4").reshape(k, dim).copy()
    nbr = np.frombuffer(take(4 * k * n), "<u4").reshape(k, n).copy()
    elen = np.frombuffer(take(4 * k * n), "<f4").reshape(k, n).copy()
    pq = np.frombuffer(take(4 * m * KSUB * dsub), "<f4").reshape(m, KSUB, dsub).copy()
    t3 = None
    if flags & FLAG_T3:
        t3 = np.frombuffer(take(4 * k * m * KSUB), "<f4").reshape(k, m, KSUB).copy()
    ncell = k * n
    off = np.zeros(ncell + 1, np.uint64)
    ids_parts, code_parts, lam_parts = [], [], []
    for c in range(ncell):
        (length,) = struct.unpack("<I", take(4))
        ids_parts.append(np.frombuffer(take(4 * length), "<u4"))
        code_parts.append(np.frombuffer(take(length * m), np.uint8))
        lam_parts.append(np.frombuffer(take(length), np.uint8))
        off[c + 1] = off[c] + length
    ids = np.concatenate(ids_parts).astype(np.uint32) if ids_parts else np.zeros(0, np.uint32)
    codes = np.concatenate(code_parts).reshape(-1, m) if code_parts else np.zeros((0, m), np.uint8)
    lams = np.concatenate(lam_parts) if lam_parts else np.zeros(0, np.uint8)
    if int(off[-1]) != count:
        raise RuntimeError("InvertedIndex: list lengths do not sum to N")
    return Vlq1(dim, k, n, m, bool(flags & FLAG_CLAMPED), lo, hi, cent, nbr, elen, pq, t3, off,
                ids, np.ascontiguousarray(codes), lams)


def write(ix: Vlq1, path: str, store_t3: bool = False) -> None:
    """serialize_index (index_io.cpp:63-98)."""
    flags = (FLAG_CLAMPED if ix.clamp else 0) | (FLAG_T3 if store_t3 else 0)
    with open(path, "wb") as f:
        f.write(b"VLQ1")
        f.write(struct.pack("<7I", 1, flags, ix.dim, ix.k, ix.n, ix.m, ix.ntotal & 0xFFFFFFFF))
        f.write(struct.pack("<2f", ix.lo, ix.hi))
        f.write(np.ascontiguousarray(ix.centroids, "<f4").tobytes())
        f.write(np.ascontiguousarray(ix.nbr, "<u4").tobytes())
        f.write(np.ascontiguousarray(ix.elen, "<f4").tobytes())
        f.write(np.ascontiguousarray(ix.pq, "<f4").tobytes())
        if store_t3:
            f.write(np.ascontiguousarray(ix.t3, "<f4").tobytes())
        off = ix.list_off
        for c in range(ix.k * ix.n):
            b0, b1 = int(off[c]), int(off[c + 1])
            f.write(struct.pack("<I", b1 - b0))
            f.write(np.ascontiguousarray(ix.ids[b0:b1], "<u4").tobytes())
            f.write(np.ascontiguousarray(ix.codes[b0:b1]).tobytes())
            f.write(np.ascontiguousarray(ix.lambdas[b0:b1]).tobytes())


def expected_size(dim: int, k: int, n: int, m: int, count: int, store_t3: bool) -> int:
    """File-size formula pinned by proj/tests/test_index.cpp:239-249."""
    return 40 + 4 * k * dim + 8 * k * n + 4 * 256 * dim + (4 * 256 * k * m if store_t3 else 0) \
        + 4 * k * n + count * (5 + m)


def read_fvecs(path: str) -> np.ndarray:
    """.fvecs reader (proj/src/vecs_io.cpp:29-86, F32 kind)."""
    raw = np.fromfile(path, dtype="<i4")
    if raw.size == 0:
        return np.zeros((0, 0), np.float32)
    d = int(raw[0])
    rec = raw.reshape(-1, d + 1)
    return rec[:, 1:].copy().view("<f4").astype(np.float32)


def write_fvecs(arr: np.ndarray, path: str) -> None:
    arr = np.ascontiguousarray(arr, np.float32)
    n, d = arr.shape
    out = np.empty((n, d + 1), "<i4")
    out[:, 0] = d
    out[:, 1:] = arr.view("<i4")
    out.tofile(path)


def read_ref_search(path: str):
    """Parses ref_tools' search output -> (ids int64[nq,k], dists f32[nq,k], scanned)."""
    with open(path, "rb") as f:
        buf = f.read()
    nq, k, scanned = struct.unpack_from("<QIQ", buf, 0)
    pos = 20
    ids = np.full((nq, k), -1, np.int64)
    dists = np.full((nq, k), np.inf, np.float32)
    for q in range(nq):
        (c,) = struct.unpack_from("<I", buf, pos)
        pos += 4
        rec = np.frombuffer(buf, "<u4", count=2 * c, offset=pos).reshape(c, 2) if c else np.zeros((0, 2), "<u4")
        pos += 8 * c
        ids[q, :c] = rec[:, 0]
        dists[q, :c] = rec[:, 1].view("<f4")
    return ids, dists, scanned


def read_ref_ivf(path: str):
    """Parses ref_tools' ivf output -> ((list_off u64[K+1], ids u32[N], codes u8[N, m]),
    (ids int64[nq,k], dists f32[nq,k], scanned))."""
    with open(path, "rb") as f:
        buf = f.read()
    K, m = struct.unpack_from("<II", buf, 0)
    pos = 8
    off = np.zeros(K + 1, np.uint64)
    ids, codes = [], []
    for c in range(K):
        (n,) = struct.unpack_from("<I", buf, pos)
        pos += 4
        ids.append(np.frombuffer(buf, "<u4", count=n, offset=pos).copy())
        pos += 4 * n
        codes.append(np.frombuffer(buf, np.uint8, count=n * m, offset=pos).reshape(n, m).copy())
        pos += n * m
        off[c + 1] = off[c] + n
    lists = (off, np.concatenate(ids).astype(np.uint32) if K else np.zeros(0, np.uint32),
             np.concatenate(codes) if K else np.zeros((0, m), np.uint8))
    nq, k, scanned = struct.unpack_from("<QIQ", buf, pos)
    pos += 20
    rid = np.full((nq, k), -1, np.int64)
    rd = np.full((nq, k), np.inf, np.float32)
    for q in range(nq):
        (c,) = struct.unpack_from("<I", buf, pos)
        pos += 4
        rec = np.frombuffer(buf, "<u4", count=2 * c, offset=pos).reshape(c, 2) if c else np.zeros((0, 2), "<u4")
        pos += 8 * c
        rid[q, :c] = rec[:, 0]
        rd[q, :c] = rec[:, 1].view("<f4")
    return lists, (rid, rd, scanned)


def file_exists(path: str) -> bool:
    return os.path.isfile(path)
