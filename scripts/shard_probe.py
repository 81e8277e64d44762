#!/usr/bin/env python
"""Per-rank cost of the select-split multi-GPU schedule, measured on ONE GPU.

Only one B200 is available to this build, so the N-GPU step is measured rank
by rank: for each (G, rank) the script builds exactly the shard that rank
would hold (lists c with shard_of_cell(c, G) == rank, coarse structures replicated), then times
with CUDA events on the GPU:

  * select   -- first_level_scan + second_level_rank for the rank's query
                slice (nq / G queries): search_select_device;
  * fine_sel -- term5 + fused scan + exact re-score for the WHOLE batch on the
                shard from the gathered selection: search_fine_sel_device;
  * merge    -- the K9 (dist, id) merge of the rank's query slice from G top-k
                blocks (vlq_group: each GPU merges its own slice);

and reports t_rank = select + fine_sel + merge.  The two all-gathers (cells +
(a, b) pairs: nq*w2*12 B; the top-k blocks: G*nq*k*12 B) are NOT measured
here (no NVLink peers); their payload sizes are printed for the model in
DESIGN.md.  The projected N-GPU batch time is the max over the sampled ranks.

  python scripts/shard_probe.py --workload c4 --shards 8:0,8:5,4:0,2:0
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="c4", choices=sorted(bench.WORKLOADS))
    ap.add_argument("--shards", default="8:0,8:5,4:0,2:0", help="comma-separated G:rank")
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--nq", type=int, default=10_000)
    ap.add_argument("--w1", type=int, default=64)
    ap.add_argument("--alpha", type=float, default=0.25)
    ap.add_argument("--k", type=int, default=100)
    ap.add_argument("--replicas", type=int, default=1,
                    help="R: the member's replica searches nq/R queries (vlq_group with N = R x S GPUs)")
    ap.add_argument("--configs", nargs="*", default=[""],
                    help="set_tuning key=value lists to time fine_sel under (first = the reported one)")
    args = ap.parse_args()
    import torch
    from paper_1901_00275_b200 import dist as vdist
    from paper_1901_00275_b200 import vlqadc
    w = bench.WORKLOADS[args.workload]
    q = bench.make_queries(vlqadc, w, args.nq, 0)
    nq, k, w1, alpha = args.nq, args.k, args.w1, args.alpha
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda:0")
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    st = stream.cuda_stream

    def timed(fn):
        for _ in range(2):
            fn()
        stream.synchronize()
        tot = 0.0
        for _ in range(args.steps):
            flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            fn()
            e1.record(stream)
            stream.synchronize()
            tot += e0.elapsed_time(e1)
        return tot / args.steps

    nq_all = nq
    nq = (nq_all + args.replicas - 1) // args.replicas  # this member's replica's part of the batch
    for spec in args.shards.split(","):
        G, rank = (int(x) for x in spec.split(":"))
        idx, setup = bench.build_index(vlqadc, w, 0, rank, G)
        w2 = idx.w2(w1, alpha)
        lo, hi = vdist.query_slice(nq, rank, G)
        sel = torch.empty((nq, w2), dtype=torch.int32, device="cuda")
        ab = torch.empty((nq, w2, 2), dtype=torch.float32, device="cuda")
        # the whole batch's selection (every rank computes its slice; here the
        # shard's replicated coarse quantizer computes all of it, untimed)
        idx.search_select_device(q.data_ptr(), nq, w1, alpha, sel.data_ptr(), ab.data_ptr(), st)
        ids = torch.empty((nq, k), dtype=torch.int64, device="cuda")
        dists = torch.empty((nq, k), dtype=torch.float32, device="cuda")
        scanned = torch.empty((nq,), dtype=torch.int64, device="cuda")
        t_sel = timed(lambda: idx.search_select_device(q[lo:hi].data_ptr(), hi - lo, w1, alpha,
                                                       sel[lo:hi].data_ptr(), ab[lo:hi].data_ptr(), st))
        idx.set_profiling(True)
        idx.stats(reset=True)
        t_fine = timed(lambda: idx.search_fine_sel_device(q.data_ptr(), nq, w1, alpha, k, sel.data_ptr(),
                                                          ab.data_ptr(), ids.data_ptr(), dists.data_ptr(),
                                                          scanned.data_ptr(), st))
        stats = idx.stats()
        idx.set_profiling(False)
        variants = {}
        ref = (ids.cpu().numpy().copy(), dists.cpu().numpy().copy())
        for cfg in args.configs[1:]:
            for kv in cfg.split(","):
                key, val = kv.split("=")
                idx.set_tuning(key, int(val))
            t = timed(lambda: idx.search_fine_sel_device(q.data_ptr(), nq, w1, alpha, k, sel.data_ptr(),
                                                         ab.data_ptr(), ids.data_ptr(), dists.data_ptr(),
                                                         scanned.data_ptr(), st))
            same = bool((ids.cpu().numpy() == ref[0]).all() and (dists.cpu().numpy() == ref[1]).all())
            variants[cfg] = {"fine_sel_ms": round(t, 3), "same_results": same}
        # the group merges only its own query slice (rows [lo, hi)) from the G blocks
        gi = ids[lo:hi].unsqueeze(0).expand(G, hi - lo, k).contiguous()
        gd = dists[lo:hi].unsqueeze(0).expand(G, hi - lo, k).contiguous()
        t_merge = timed(lambda: vdist.merge_topk(gi, gd, st))
        # the earlier schedule for comparison: query-split first level only,
        # every rank repeats exact neighbours + second level for the batch
        top = torch.empty((nq, w1), dtype=torch.int32, device="cuda")
        idx.search_coarse_device(q.data_ptr(), nq, w1, top.data_ptr(), st)
        t_coarse = timed(lambda: idx.search_coarse_device(q[lo:hi].data_ptr(), hi - lo, w1, top[lo:hi].data_ptr(),
                                                          st))
        t_fine_top = timed(lambda: idx.search_fine_device(q.data_ptr(), nq, w1, alpha, k, top.data_ptr(),
                                                          ids.data_ptr(), dists.data_ptr(), scanned.data_ptr(), st))
        steps = args.steps + 2  # timed() runs 2 warm-up calls inside the profiled window
        line = {"workload": args.workload, "G": G, "rank": rank, "replicas": args.replicas, "nq_batch": nq_all,
                "nq": nq, "w1": w1, "alpha": alpha, "k": k,
                "local_entries": idx.local_entries,
                "scanned_local_per_query": round(float(scanned.sum().item()) / nq, 1),
                "select_split_ms": {"select_slice": round(t_sel, 3), "fine_sel": round(t_fine, 3),
                                    "merge": round(t_merge, 3),
                                    "rank_total_excl_collectives": round(t_sel + t_fine + t_merge, 3)},
                "query_split_ms": {"coarse_slice": round(t_coarse, 3), "fine": round(t_fine_top, 3),
                                   "merge": round(t_merge, 3),
                                   "rank_total_excl_collectives": round(t_coarse + t_fine_top + t_merge, 3)},
                "fine_sel_phase_ms": {p: round(v / steps, 4) for p, v in stats["phase_ms"].items()},
                "fine_sel_variants": variants,
                "collective_bytes": {"selection_allgather_per_rank": nq * w2 * 12,
                                     "topk_allgather_per_rank": G * nq * k * 12},
                "l2": "flushed before every timed call", "setup": setup}
        print(json.dumps(line), flush=True)
        del idx
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
