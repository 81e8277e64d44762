"""CPU test of the multi-GPU path's host logic (gloo, world_size 2).

Each rank holds the posting lists c with shard_of_cell(c, world) == rank of the
golden index (the engine's shard rule, csrc/engine.h), searches its shard, and the
per-shard top-k blocks are exchanged with paper_1901_00275_b200.dist.gather_parts
(the same call the NCCL path uses).  The (dist, id) merge of the gathered
blocks must equal the unsharded search.  The shard search and the merge here
are the oracle's (no GPU on this box); the GPU merge kernel is covered by
tests/test_gpu_parity.py::test_sharded_engines_merge_to_the_single_engine_result.
"""
import os
import socket

import numpy as np
import pytest

from conftest import ROOT, load_golden


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def shard_of_cell(c, shards):
    """The engine's list ownership (csrc/engine.h shard_of_cell)."""
    return (((c * 0x9E3779B97F4A7C15) & ((1 << 64) - 1)) >> 40) % shards


def shard_of(ix, rank, world):
    from oracle import vlq1
    keep = np.zeros(ix.k * ix.n, bool)
    for c in range(ix.k * ix.n):
        keep[c] = shard_of_cell(c, world) == rank
    lens = np.diff(ix.list_off.astype(np.int64))
    lens = np.where(keep, lens, 0)
    off = np.zeros(ix.k * ix.n + 1, np.uint64)
    np.cumsum(lens, out=off[1:])
    sel = np.concatenate([np.arange(int(ix.list_off[c]), int(ix.list_off[c + 1])) for c in range(ix.k * ix.n)
                          if keep[c]] or [np.zeros(0, np.int64)]).astype(np.int64)
    return vlq1.Vlq1(ix.dim, ix.k, ix.n, ix.m, ix.clamp, ix.lo, ix.hi, ix.centroids, ix.nbr, ix.elen, ix.pq, ix.t3, off,
                     ix.ids[sel], ix.codes[sel], ix.lambdas[sel])


def merge_np(ids, dists):
    """(dist, id) merge of [G, nq, k] blocks, -1/inf padded (the K9 contract)."""
    G, nq, k = ids.shape
    out_i = np.full((nq, k), -1, np.int64)
    out_d = np.full((nq, k), np.inf, np.float32)
    for q in range(nq):
        cand = [(float(dists[g, q, j]), int(ids[g, q, j])) for g in range(G) for j in range(k) if ids[g, q, j] >= 0]
        cand.sort()
        for j, (d, i) in enumerate(cand[:k]):
            out_i[q, j], out_d[q, j] = i, d
    return out_i, out_d


def _worker(rank, world, port, name, params, out_path):
    import sys
    sys.path.insert(0, ROOT)
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import oracle, vlq1
    from paper_1901_00275_b200.dist import gather_parts
    z, index_path, _ = load_golden(name)
    ix = vlq1.read(index_path)
    o = oracle.OracleIndex(shard_of(ix, rank, world))
    res = []
    for w1, alpha, k in params:
        ids, d, _ = o.search(z["queries"], w1, alpha, k)
        gi, gd = gather_parts(torch.from_numpy(ids), torch.from_numpy(d))
        res.append((gi.numpy(), gd.numpy()))
    if rank == 0:
        import pickle
        with open(out_path, "wb") as f:
            pickle.dump([merge_np(*r) for r in res], f)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("name", ["accept_small", "m16"])
def test_gloo_sharded_search_merges_to_single_index(name, tmp_path):
    import torch.multiprocessing as mp
    from oracle import oracle
    params = [(16, 0.5, 10), (64, 0.25, 100), (4, 1.0, 7)]
    out = str(tmp_path / "merged.pkl")
    mp.start_processes(_worker, args=(2, _free_port(), name, params, out), nprocs=2, join=True, start_method="spawn")
    import pickle
    with open(out, "rb") as f:
        merged = pickle.load(f)
    z, index_path, _ = load_golden(name)
    o = oracle.OracleIndex.load(index_path)
    for (w1, alpha, k), (mi, md) in zip(params, merged):
        ids, d, _ = o.search(z["queries"], w1, alpha, k)
        assert np.array_equal(mi, ids)
        assert np.array_equal(np.asarray(md, np.float32).view(np.uint32), d.view(np.uint32))


def _worker_query_split(rank, world, port, name, params, out_path):
    """The query-split schedule of ShardedIndex.search_query_split with the
    oracle standing in for the engine: coarse stage on this rank's query
    slice only, all-gather of the top-w1 tables (dist.gather_top), fine stage
    for the whole batch on this rank's shard, all-gather of the top-k blocks."""
    import sys
    sys.path.insert(0, ROOT)
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import oracle, vlq1
    from paper_1901_00275_b200.dist import gather_parts, gather_top, query_slice
    z, index_path, _ = load_golden(name)
    ix = vlq1.read(index_path)
    full = oracle.OracleIndex(ix)                      # the replicated coarse quantizer
    shard = oracle.OracleIndex(shard_of(ix, rank, world))
    q = z["queries"]
    res = []
    for w1, alpha, k in params:
        lo, hi = query_slice(q.shape[0], rank, world)
        top_local = torch.from_numpy(full.first_level(q[lo:hi], w1).view(np.int32))
        top = gather_top(top_local, q.shape[0], w1).numpy().view(np.uint32)
        ids, d, _ = shard.search_from_top(q, top, w1, alpha, k)
        gi, gd = gather_parts(torch.from_numpy(ids), torch.from_numpy(d))
        res.append((gi.numpy(), gd.numpy()))
    if rank == 0:
        import pickle
        with open(out_path, "wb") as f:
            pickle.dump([merge_np(*r) for r in res], f)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_gloo_query_split_coarse_stage_merges_to_single_index(world, tmp_path):
    import torch.multiprocessing as mp
    from oracle import oracle
    name = "accept_small"
    params = [(16, 0.5, 10), (64, 0.25, 100), (3, 1.0, 5)]
    out = str(tmp_path / "merged.pkl")
    mp.start_processes(_worker_query_split, args=(world, _free_port(), name, params, out), nprocs=world, join=True,
                       start_method="spawn")
    import pickle
    with open(out, "rb") as f:
        merged = pickle.load(f)
    z, index_path, _ = load_golden(name)
    o = oracle.OracleIndex.load(index_path)
    for (w1, alpha, k), (mi, md) in zip(params, merged):
        ids, d, _ = o.search(z["queries"], w1, alpha, k)
        assert np.array_equal(mi, ids)
        assert np.array_equal(np.asarray(md, np.float32).view(np.uint32), d.view(np.uint32))


def _worker_select_split(rank, world, port, name, params, out_path):
    """The select-split schedule of ShardedIndex.search_select_split with the
    oracle standing in for the engine: first level + cell selection on this
    rank's query slice only, all-gather of the selected cells and their
    (a, b) pairs (dist.gather_rows), scan stage for the whole batch on this
    rank's shard starting from the hand-off alone, all-gather of the top-k
    blocks."""
    import sys
    sys.path.insert(0, ROOT)
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import oracle, vlq1
    from paper_1901_00275_b200.dist import gather_parts, gather_rows, query_slice
    z, index_path, _ = load_golden(name)
    ix = vlq1.read(index_path)
    full = oracle.OracleIndex(ix)                      # the replicated coarse quantizer
    shard = oracle.OracleIndex(shard_of(ix, rank, world))
    q = z["queries"]
    res = []
    for w1, alpha, k in params:
        lo, hi = query_slice(q.shape[0], rank, world)
        sel_l, ab_l = full.select(q[lo:hi], w1, alpha)
        sel = gather_rows(torch.from_numpy(sel_l.view(np.int32)), q.shape[0]).numpy().view(np.uint32)
        ab = gather_rows(torch.from_numpy(ab_l), q.shape[0]).numpy()
        ids, d, _ = shard.search_from_sel(q, sel, ab, w1, alpha, k)
        gi, gd = gather_parts(torch.from_numpy(ids), torch.from_numpy(d))
        res.append((gi.numpy(), gd.numpy()))
    if rank == 0:
        import pickle
        with open(out_path, "wb") as f:
            pickle.dump([merge_np(*r) for r in res], f)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_gloo_select_split_merges_to_single_index(world, tmp_path):
    import torch.multiprocessing as mp
    from oracle import oracle
    name = "accept_small"
    params = [(16, 0.5, 10), (64, 0.25, 100), (3, 1.0, 5)]
    out = str(tmp_path / "merged.pkl")
    mp.start_processes(_worker_select_split, args=(world, _free_port(), name, params, out), nprocs=world, join=True,
                       start_method="spawn")
    import pickle
    with open(out, "rb") as f:
        merged = pickle.load(f)
    z, index_path, _ = load_golden(name)
    o = oracle.OracleIndex.load(index_path)
    for (w1, alpha, k), (mi, md) in zip(params, merged):
        ids, d, _ = o.search(z["queries"], w1, alpha, k)
        assert np.array_equal(mi, ids)
        assert np.array_equal(np.asarray(md, np.float32).view(np.uint32), d.view(np.uint32))


def test_oracle_select_split_equals_search():
    """select() + search_from_sel() (the hand-off alone: the scan stage sees
    only the selected cells and their a, b) equals search()."""
    from oracle import oracle
    for name in ("m16", "accept_small"):
        z, index_path, _ = load_golden(name)
        o = oracle.OracleIndex.load(index_path)
        q = z["queries"]
        for w1, alpha, k in [(8, 0.5, 10), (32, 0.25, 100), (o.ix.k, 1.0, 7)]:
            sel, ab = o.select(q, w1, alpha)
            a = o.search(q, w1, alpha, k)
            b = o.search_from_sel(q, sel, ab, w1, alpha, k)
            for x, y in zip(a, b):
                assert np.array_equal(x, y)


def test_query_slices_cover_the_batch():
    from paper_1901_00275_b200.dist import query_slice
    for nq in (0, 1, 7, 100, 10_000):
        for world in (1, 2, 3, 8):
            cover = []
            for r in range(world):
                lo, hi = query_slice(nq, r, world)
                assert 0 <= lo <= hi <= nq
                cover.extend(range(lo, hi))
            assert cover == list(range(nq))


def test_oracle_staged_search_equals_search():
    from oracle import oracle
    z, index_path, _ = load_golden("m16")
    o = oracle.OracleIndex.load(index_path)
    q = z["queries"]
    for w1, alpha, k in [(8, 0.5, 10), (32, 0.25, 100)]:
        top = o.first_level(q, w1)
        a = o.search(q, w1, alpha, k)
        b = o.search_from_top(q, top, w1, alpha, k)
        for x, y in zip(a, b):
            assert np.array_equal(x, y)


def test_shard_of_cell_matches_the_engine():
    """The Python restatement used by these tests == the engine's ownership
    function (exported by libvlqgpu.so; host-only, no GPU needed), and the
    hash spreads a region's n lists and the lists overall evenly."""
    from paper_1901_00275_b200 import _lib
    L = _lib.lib()
    rng = np.random.default_rng(7)
    cells = np.concatenate([np.arange(4096), rng.integers(0, 2**31, 4096)])
    for shards in (1, 2, 3, 4, 8):
        got = np.array([L.vlq_shard_of_cell(int(c), shards) for c in cells])
        want = np.array([shard_of_cell(int(c), shards) for c in cells])
        assert np.array_equal(got, want)
    counts = np.bincount([shard_of_cell(c, 8) for c in range(65536 * 32)], minlength=8)
    assert counts.min() > 0.99 * counts.mean() and counts.max() < 1.01 * counts.mean()
    region = [shard_of_cell(17 * 32 + j, 8) for j in range(32)]
    assert len(set(region)) >= 6  # one region's lists land on most ranks


def _worker_slice_merge(rank, world, port, name, params, out_path):
    """dist.slice_merge (the select-split schedule's merge by query slice:
    all-to-all of the slices' rows, per-rank merge of its slice, all-gather of
    the merged slices) over oracle shard results."""
    import sys
    sys.path.insert(0, ROOT)
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import oracle, vlq1
    from paper_1901_00275_b200.dist import slice_merge
    z, index_path, _ = load_golden(name)
    ix = vlq1.read(index_path)
    shard = oracle.OracleIndex(shard_of(ix, rank, world))

    def np_merge(pi, pd):
        mi, md = merge_np(pi.numpy(), pd.numpy())
        return torch.from_numpy(mi), torch.from_numpy(md)

    res = []
    for w1, alpha, k in params:
        ids, d, _ = shard.search(z["queries"], w1, alpha, k)
        mi, md = slice_merge(torch.from_numpy(ids), torch.from_numpy(d), merge_fn=np_merge)
        res.append((mi.numpy(), md.numpy()))
    if rank == 0:
        import pickle
        with open(out_path, "wb") as f:
            pickle.dump(res, f)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_gloo_slice_merge_equals_single_index(world, tmp_path):
    import torch.multiprocessing as mp
    from oracle import oracle
    name = "accept_small"
    params = [(16, 0.5, 10), (64, 0.25, 100)]
    out = str(tmp_path / "merged.pkl")
    mp.start_processes(_worker_slice_merge, args=(world, _free_port(), name, params, out), nprocs=world, join=True,
                       start_method="spawn")
    import pickle
    with open(out, "rb") as f:
        merged = pickle.load(f)
    z, index_path, _ = load_golden(name)
    o = oracle.OracleIndex.load(index_path)
    for (w1, alpha, k), (mi, md) in zip(params, merged):
        ids, d, _ = o.search(z["queries"], w1, alpha, k)
        assert np.array_equal(mi, ids)
        assert np.array_equal(np.asarray(md, np.float32).view(np.uint32), d.view(np.uint32))
