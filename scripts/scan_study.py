#!/usr/bin/env python
"""A/B study of search-kernel variants on ONE built index (GPU box only).

Builds the workload's index once (as bench.py does), then for every
configuration times `--steps` batched searches with per-phase CUDA events and
checks that the results equal the first configuration's bit for bit.

  python scripts/scan_study.py --workload c4 --configs "scan_slots=6" "scan_slots=104"
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
    ap.add_argument("--workload", default="c4", choices=sorted(bench.WORKLOADS))
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--nq", type=int, default=10_000)
    ap.add_argument("--w1", type=int, default=64)
    ap.add_argument("--alpha", type=float, default=0.25)
    ap.add_argument("--k", type=int, default=100)
    ap.add_argument("--configs", nargs="+", default=["scan_slots=0"])
    ap.add_argument("--hubs", action="store_true", help="region-visit skew: bytes of the hottest regions vs reads")
    args = ap.parse_args()
    import torch
    from paper_1901_00275_b200 import vlqadc
    w = bench.WORKLOADS[args.workload]
    idx, setup = bench.build_index(vlqadc, w, 0)
    q = bench.make_queries(vlqadc, w, args.nq, 0)
    nq, k = args.nq, args.k
    ids = torch.empty((nq, k), dtype=torch.int64, device=q.device)
    dists = torch.empty((nq, k), dtype=torch.float32, device=q.device)
    scanned = torch.empty((nq,), dtype=torch.int64, device=q.device)
    flush = torch.empty(512 << 20, dtype=torch.uint8, device=q.device)
    st = torch.cuda.current_stream().cuda_stream
    if args.hubs:
        top = torch.empty((nq, args.w1), dtype=torch.int32, device=q.device)
        idx.search_coarse_device(q.data_ptr(), nq, args.w1, top.data_ptr(), st)
        torch.cuda.synchronize()
        visits = np.bincount(top.cpu().numpy().ravel().view(np.uint32), minlength=w["k"]).astype(np.float64)
        off = idx.list_offsets().astype(np.int64)
        nreg = w["k"]
        rb = (off[np.arange(1, nreg + 1) * w["edges"]] - off[np.arange(nreg) * w["edges"]]) * (w["m"] + 5)
        order = np.argsort(-visits, kind="stable")
        cb = np.cumsum(rb[order])
        cr = np.cumsum((visits * rb)[order])
        out = {"regions_visited": int((visits > 0).sum()), "mean_visits": float(visits.mean()),
               "max_visits": int(visits.max()), "region_reads_gb": float(cr[-1] / 1e9)}
        for mb in (32, 64, 96, 128, 512, 2048):
            j = int(np.searchsorted(cb, mb * 1e6))
            out[f"reads_in_hottest_{mb}MB"] = round(float(cr[min(j, len(cr) - 1)] / cr[-1]), 4)
        print(json.dumps({"hubs": out}), flush=True)
    ref = None
    for cfg in args.configs:
        clk = bench.ClockSampler(0)
        for kv in cfg.split(","):
            key, val = kv.split("=")
            idx.set_tuning(key, int(val))
        for _ in range(2):
            idx.search_device(q.data_ptr(), nq, args.w1, args.alpha, k, ids.data_ptr(), dists.data_ptr(),
                              scanned.data_ptr(), st)
        idx.sync(st)
        idx.set_profiling(True)
        idx.stats(reset=True)
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        tot = 0.0
        with clk:
            for _ in range(args.steps):
                flush.zero_()
                ev0.record()
                idx.search_device(q.data_ptr(), nq, args.w1, args.alpha, k, ids.data_ptr(), dists.data_ptr(),
                                  scanned.data_ptr(), st)
                ev1.record()
                torch.cuda.synchronize()
                tot += ev0.elapsed_time(ev1)
        stats = idx.stats()
        idx.set_profiling(False)
        res = (ids.cpu().numpy().copy(), dists.cpu().numpy().view(np.uint32).copy())
        same = None
        if ref is None:
            ref = res
        else:
            same = bool(np.array_equal(res[0], ref[0]) and np.array_equal(res[1], ref[1]))
        sc = int(scanned.sum().item())
        scan_ms = stats["phase_ms"]["scan"] / args.steps
        line = {"workload": args.workload, "config": cfg, "ms_per_step": round(tot / args.steps, 3),
                "qps": round(nq * args.steps / (tot / 1e3), 1),
                "phase_ms": {p: round(v / args.steps, 3) for p, v in stats["phase_ms"].items()},
                "scan_gbs": round(sc * (w["m"] + 5) / (scan_ms / 1e3) / 1e9, 1) if scan_ms else None,
                "flagged_per_step": stats["flagged"] / args.steps, "clocks": clk.summary(),
                "same_as_first": same, "setup": setup}
        print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
