"""Multi-GPU search: posting lists sharded by first-level region across the GPUs
of one box (one process per GPU), coarse quantizer replicated, per-shard
top-k merged by (dist, id) (the paper's "split the index into b parts, search
locally, join").

Each rank's engine holds the posting lists (cells) c with
((c * 0x9E3779B97F4A7C15) mod 2^64 >> 40) % world_size == rank (csrc/engine.h
shard_of_cell: a hash, so every region's n lists and every hub region spread
over all ranks).  Per batch
(`ShardedIndex.search_select_split`, the default schedule):

1. query-split selection: rank r runs first_level_scan (the tensor-core GEMM
   + exact refine, search.cpp:11-36) AND second_level_rank (search.cpp:38-78)
   for its slice of the batch only -- everything whose cost does not shrink
   with the shard;
2. the slices' selections are exchanged with two NCCL all-gathers: the
   selected cells (nq x w2 u32, 20 MB at nq = 10k, w2 = 512) and their exact
   (a, b) = (|y - c_i|^2, |y - c_nbr|^2) pairs (41 MB), the only coarse values
   the later stages read;
3. every rank applies the gathered selection (its own scanned counts and
   certificate bound) and runs term5, the fused scan and the exact re-score
   for the whole batch on the cells it owns;
4. the local exact top-k rows are exchanged BY QUERY SLICE (one all-to-all:
   rank r receives every rank's rows of its slice), each rank merges its own
   slice with the K9 kernel (vlq_merge_topk_device), and the merged slices
   are all-gathered (slice_merge).

`search_query_split` is the earlier schedule: only first_level_scan is split
(top-w1 tables, 2.5 MB, all-gathered) and every rank repeats the exact
neighbour distances and second_level_rank for the whole batch.

Because every shard returns its exact local top-k under the reference's total
order, the merge is exactly the single-engine answer regardless of shard
order (both schedules).
"""
from __future__ import annotations

import ctypes

from . import _lib


def merge_topk(ids, dists, stream: int | None = None):
    """ids int64 [G, nq, k], dists float32 [G, nq, k] (CUDA tensors) -> the
    merged (nq, k) top-k under (dist, id)."""
    import torch
    G, nq, k = ids.shape
    ids = ids.contiguous()
    dists = dists.contiguous()
    out_i = torch.empty((nq, k), dtype=torch.int64, device=ids.device)
    out_d = torch.empty((nq, k), dtype=torch.float32, device=ids.device)
    st = torch.cuda.current_stream(ids.device).cuda_stream if stream is None else stream
    _lib.check(_lib.lib().vlq_merge_topk_device(ids.device.index, ctypes.c_void_p(ids.data_ptr()),
                                                ctypes.c_void_p(dists.data_ptr()), G, nq, k,
                                                ctypes.c_void_p(out_i.data_ptr()), ctypes.c_void_p(out_d.data_ptr()),
                                                ctypes.c_void_p(st)))
    return out_i, out_d


def _all_gather(out, inp, group=None):
    """all_gather_into_tensor; CUDA tensors go through host copies when the
    backend cannot take them (gloo: the single-GPU rehearsal of N > 1)."""
    import torch.distributed as dist
    if inp.is_cuda and dist.get_backend(group) != "nccl":
        o = out.cpu()
        dist.all_gather_into_tensor(o, inp.cpu(), group=group)
        out.copy_(o)
    else:
        dist.all_gather_into_tensor(out, inp, group=group)


def gather_parts(local_ids, local_dists, group=None):
    """All-gathers every rank's [nq, k] result block into [world, nq, k]."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    nq = local_ids.shape[0]
    # concatenated along dim 0 (the layout every backend accepts), viewed [world, nq, k]
    gi = torch.empty((world * nq,) + tuple(local_ids.shape[1:]), dtype=local_ids.dtype, device=local_ids.device)
    gd = torch.empty((world * nq,) + tuple(local_dists.shape[1:]), dtype=local_dists.dtype, device=local_dists.device)
    _all_gather(gi, local_ids.contiguous(), group)
    _all_gather(gd, local_dists.contiguous(), group)
    return gi.view((world,) + tuple(local_ids.shape)), gd.view((world,) + tuple(local_dists.shape))


def _all_to_all(out, inp, group=None):
    """all_to_all_single over equal row blocks (host copies for gloo)."""
    import torch.distributed as dist
    if inp.is_cuda and dist.get_backend(group) != "nccl":
        o = out.cpu()
        dist.all_to_all_single(o, inp.cpu(), group=group)
        out.copy_(o)
    else:
        dist.all_to_all_single(out, inp, group=group)


def slice_merge(local_ids, local_dists, group=None, merge_fn=None):
    """(dist, id) merge of the per-shard top-k blocks BY QUERY SLICE: rank r
    receives the rows of its slice (query_slice) from every rank (one
    all-to-all: nq/G x k x 12 bytes from each peer instead of the whole
    blocks), merges only those, and the merged slices are all-gathered.
    Returns the merged [nq, k] (ids, dists) on every rank.  merge_fn(ids [G,
    rows, k], dists) -> merged; default: the K9 kernel (merge_topk)."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    nq, k = local_ids.shape
    per = (nq + world - 1) // world
    si = torch.full((world * per, k), -1, dtype=local_ids.dtype, device=local_ids.device)
    sd = torch.full((world * per, k), float("inf"), dtype=local_dists.dtype, device=local_dists.device)
    si[:nq] = local_ids
    sd[:nq] = local_dists
    ri, rd = torch.empty_like(si), torch.empty_like(sd)
    _all_to_all(ri, si, group)
    _all_to_all(rd, sd, group)
    parts_i, parts_d = ri.view(world, per, k), rd.view(world, per, k)
    mi, md = (merge_fn or merge_topk)(parts_i, parts_d)
    return gather_rows(mi, nq, group), gather_rows(md, nq, group)


def query_slice(nq: int, rank: int, world: int) -> tuple[int, int]:
    """Rows [lo, hi) of an nq-query batch whose coarse stage rank runs (equal
    ceil-sized slices; the last ones may be short or empty)."""
    per = (nq + world - 1) // world
    lo = min(nq, rank * per)
    return lo, min(nq, lo + per)


def gather_top(local_top, nq: int, w1: int, group=None):
    """All-gathers every rank's [slice, w1] top-w1 block into the [nq, w1]
    table (slices padded to the common ceil size for the collective)."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    per = (nq + world - 1) // world
    send = torch.zeros((per, w1), dtype=local_top.dtype, device=local_top.device)
    send[:local_top.shape[0]] = local_top
    out = torch.empty((world * per, w1), dtype=local_top.dtype, device=local_top.device)
    _all_gather(out, send, group)
    return out[:nq]


def gather_rows(local, nq: int, group=None):
    """All-gathers every rank's [slice, ...] block (query_slice rows) into the
    [nq, ...] batch table (slices padded to the common ceil size)."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    per = (nq + world - 1) // world
    tail = tuple(local.shape[1:])
    send = torch.zeros((per,) + tail, dtype=local.dtype, device=local.device)
    send[:local.shape[0]] = local
    out = torch.empty((world * per,) + tail, dtype=local.dtype, device=local.device)
    _all_gather(out, send, group)
    return out[:nq]


class ShardedIndex:
    """One rank's shard of a VLQ1 index plus the collective search."""

    def __init__(self, index, group=None):
        self.index = index
        self.group = group

    @classmethod
    def load(cls, path: str, rank: int, world: int, device: int, group=None, **kw):
        from .vlqadc import Index
        return cls(Index.load(path, device=device, shard_rank=rank, shard_count=world, **kw), group)

    def search_device(self, d_queries, w1: int, alpha: float, k: int):
        """d_queries: CUDA float32 [nq, dim] tensor (same batch on every rank).
        Returns the merged (ids, dists) CUDA tensors and the local scanned
        counts."""
        import torch
        nq = d_queries.shape[0]
        dev = d_queries.device
        ids = torch.empty((nq, k), dtype=torch.int64, device=dev)
        dists = torch.empty((nq, k), dtype=torch.float32, device=dev)
        scanned = torch.empty((nq,), dtype=torch.int64, device=dev)
        st = torch.cuda.current_stream(dev).cuda_stream
        self.index.search_device(d_queries.data_ptr(), nq, w1, alpha, k, ids.data_ptr(), dists.data_ptr(),
                                 scanned.data_ptr(), st)
        gi, gd = gather_parts(ids, dists, self.group)
        mi, md = merge_topk(gi, gd, st)
        return mi, md, scanned

    def search_query_split(self, d_queries, w1: int, alpha: float, k: int, out=None):
        """Query-split coarse stage + sharded fine stage (module docstring).
        d_queries: the same CUDA float32 [nq, dim] batch on every rank.
        Returns the merged (ids, dists) and the local scanned counts."""
        import torch
        import torch.distributed as dist
        nq = d_queries.shape[0]
        dev = d_queries.device
        rank, world = dist.get_rank(self.group), dist.get_world_size(self.group)
        st = torch.cuda.current_stream(dev).cuda_stream
        lo, hi = query_slice(nq, rank, world)
        top_local = torch.empty((hi - lo, w1), dtype=torch.int32, device=dev)
        if hi > lo:
            self.index.search_coarse_device(d_queries[lo:hi].data_ptr(), hi - lo, w1, top_local.data_ptr(), st)
        top = gather_top(top_local, nq, w1, self.group).contiguous()
        if out is None:
            out = (torch.empty((nq, k), dtype=torch.int64, device=dev),
                   torch.empty((nq, k), dtype=torch.float32, device=dev),
                   torch.empty((nq,), dtype=torch.int64, device=dev))
        ids, dists, scanned = out
        self.index.search_fine_device(d_queries.data_ptr(), nq, w1, alpha, k, top.data_ptr(), ids.data_ptr(),
                                      dists.data_ptr(), scanned.data_ptr(), st)
        gi, gd = gather_parts(ids, dists, self.group)
        mi, md = merge_topk(gi, gd, st)
        return mi, md, scanned

    def search_select_split(self, d_queries, w1: int, alpha: float, k: int, out=None):
        """Query-split coarse stage and cell selection + sharded scan stage
        (module docstring).  d_queries: the same CUDA float32 [nq, dim] batch
        on every rank.  Returns the merged (ids, dists) and the local scanned
        counts."""
        import torch
        import torch.distributed as dist
        nq = d_queries.shape[0]
        dev = d_queries.device
        rank, world = dist.get_rank(self.group), dist.get_world_size(self.group)
        st = torch.cuda.current_stream(dev).cuda_stream
        w2 = self.index.w2(w1, alpha)
        lo, hi = query_slice(nq, rank, world)
        sel_local = torch.empty((hi - lo, w2), dtype=torch.int32, device=dev)
        ab_local = torch.empty((hi - lo, w2, 2), dtype=torch.float32, device=dev)
        if hi > lo:
            self.index.search_select_device(d_queries[lo:hi].data_ptr(), hi - lo, w1, alpha, sel_local.data_ptr(),
                                            ab_local.data_ptr(), st)
        sel = gather_rows(sel_local, nq, self.group).contiguous()
        ab = gather_rows(ab_local, nq, self.group).contiguous()
        if out is None:
            out = (torch.empty((nq, k), dtype=torch.int64, device=dev),
                   torch.empty((nq, k), dtype=torch.float32, device=dev),
                   torch.empty((nq,), dtype=torch.int64, device=dev))
        ids, dists, scanned = out
        self.index.search_fine_sel_device(d_queries.data_ptr(), nq, w1, alpha, k, sel.data_ptr(), ab.data_ptr(),
                                          ids.data_ptr(), dists.data_ptr(), scanned.data_ptr(), st)
        # merge by query slice: all-to-all of the slices' rows, each rank merges
        # its own slice, the merged slices are all-gathered
        mi, md = slice_merge(ids, dists, self.group, lambda pi, pd: merge_topk(pi, pd, st))
        return mi, md, scanned
