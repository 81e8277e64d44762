#!/usr/bin/env python
"""QPS-recall curve on ONE built index (GPU box only): BASELINE.json configs[4]
("QPS-recall@1/10/100 curve at query batch 1k/10k/100k") on one B200.

Builds the workload's index once (as bench.py does), then for every query
batch size and w1 times `--steps` device-resident batched searches (CUDA
events, L2 flushed between steps) and scores recall@1/10/100 against the
exact ground truth of the first `--gt` queries (GPU brute force, eval.cpp:
13-36 semantics).  One JSON line per (nq, w1).

  python scripts/curve.py --workload c5 --nqs 1000,10000,100000 --w1s 16,32,64,128
"""
import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="c5", choices=sorted(bench.WORKLOADS))
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--nqs", default="1000,10000,100000")
    ap.add_argument("--w1s", default="16,32,64,128")
    ap.add_argument("--alpha", type=float, default=0.25)
    ap.add_argument("--k", type=int, default=100)
    ap.add_argument("--gt", type=int, default=200)
    ap.add_argument("--queries", default="ref,heldout", help="query sets: ref (reference convention), heldout")
    args = ap.parse_args()
    import torch
    from paper_1901_00275_b200 import vlqadc
    w = bench.WORKLOADS[args.workload]
    idx, setup = bench.build_index(vlqadc, w, 0)
    nqs = [int(x) for x in args.nqs.split(",") if x]
    w1s = [int(x) for x in args.w1s.split(",") if x]
    k = args.k
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda:0")
    stream = torch.cuda.Stream()
    st = stream.cuda_stream
    for kind in [x for x in args.queries.split(",") if x]:
        qall = bench.make_queries(vlqadc, w, max(nqs), 0, kind=kind)
        ngt = min(args.gt, min(nqs))
        gt = vlqadc.brute_force_gt_synthetic(w["n"], w["dim"], w["clusters"], bench.SPREAD, bench.BASE_SEED,
                                             qall[:ngt].cpu().numpy(), 1, device=0)
        run(args, idx, qall, nqs, w1s, k, gt, ngt, flush, stream, st, setup, kind)


def run(args, idx, qall, nqs, w1s, k, gt, ngt, flush, stream, st, setup, kind):
    import torch
    for nq in nqs:
        q = qall[:nq].contiguous()
        ids = torch.empty((nq, k), dtype=torch.int64, device=q.device)
        dists = torch.empty((nq, k), dtype=torch.float32, device=q.device)
        scanned = torch.empty((nq,), dtype=torch.int64, device=q.device)
        for w1 in w1s:
            clk = bench.ClockSampler(0)
            torch.cuda.synchronize()
            with torch.cuda.stream(stream):
                for _ in range(3):
                    idx.search_device(q.data_ptr(), nq, w1, args.alpha, k, ids.data_ptr(), dists.data_ptr(),
                                      scanned.data_ptr(), st)
                stream.synchronize()
                tot = 0.0
                with clk:
                    for _ in range(args.steps):
                        flush.zero_()
                        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                        e0.record(stream)
                        idx.search_device(q.data_ptr(), nq, w1, args.alpha, k, ids.data_ptr(), dists.data_ptr(),
                                          scanned.data_ptr(), st)
                        e1.record(stream)
                        stream.synchronize()
                        tot += e0.elapsed_time(e1)
            res = ids[:ngt].cpu().numpy()
            line = {"workload": args.workload, "queries": kind, "nq": nq, "w1": w1, "alpha": args.alpha, "k": k,
                    "qps": round(nq * args.steps / (tot / 1e3), 1), "ms_per_step": round(tot / args.steps, 3),
                    "scanned_per_query": round(float(scanned.sum().item()) / nq, 1),
                    **{f"recall@{r}": round(bench.recall_at(res, gt, r), 4) for r in (1, 10, 100) if r <= k},
                    "gt_queries": ngt, "l2": "flushed between steps (512 MiB write)", "clocks": clk.summary(),
                    "setup": setup}
            print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
