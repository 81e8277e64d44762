#!/usr/bin/env python
"""Where the end-to-end (host numpy in/out) search time goes beyond the
device-timed search: times, on one built index, the device-resident search
(CUDA events), the public Index.search on numpy arrays (wall clock), and the
host<->device traffic of one call alone (pinned copies, and the pageable
numpy copies the API performs).

  python scripts/e2e_probe.py --workload c2
"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="c2", choices=sorted(bench.WORKLOADS))
    ap.add_argument("--nq", type=int, default=10_000)
    ap.add_argument("--k", type=int, default=100)
    ap.add_argument("--reps", type=int, default=10)
    args = ap.parse_args()
    import torch
    from paper_1901_00275_b200 import vlqadc
    w = bench.WORKLOADS[args.workload]
    idx, _ = bench.build_index(vlqadc, w, 0)
    q = bench.make_queries(vlqadc, w, args.nq, 0)
    qh = q.cpu().numpy()
    nq, k = args.nq, args.k
    ids = torch.empty((nq, k), dtype=torch.int64, device="cuda")
    dists = torch.empty((nq, k), dtype=torch.float32, device="cuda")
    st = torch.cuda.current_stream().cuda_stream
    out = {"workload": args.workload, "nq": nq, "k": k}
    for _ in range(3):
        idx.search_device(q.data_ptr(), nq, 64, 0.25, k, ids.data_ptr(), dists.data_ptr(), None, st)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(args.reps):
        idx.search_device(q.data_ptr(), nq, 64, 0.25, k, ids.data_ptr(), dists.data_ptr(), None, st)
    e1.record()
    torch.cuda.synchronize()
    out["device_ms"] = round(e0.elapsed_time(e1) / args.reps, 3)
    idx.search(qh, w1=64, alpha=0.25, k=k)
    t = []
    for _ in range(args.reps):
        t0 = time.perf_counter()
        idx.search(qh, w1=64, alpha=0.25, k=k)
        t.append(time.perf_counter() - t0)
    out["host_api_ms"] = round(1e3 * float(np.median(t)), 3)
    # the bare C call on preallocated outputs (no Python-side allocation)
    import ctypes
    from paper_1901_00275_b200 import _lib
    oi = np.empty((nq, k), np.int64)
    od = np.empty((nq, k), np.float32)
    osc = np.empty(nq, np.uint64)
    t = []
    for _ in range(args.reps):
        t0 = time.perf_counter()
        _lib.check(_lib.lib().vlq_engine_search(idx._h, qh.ctypes.data_as(ctypes.c_void_p), nq, qh.shape[1], 64,
                                                0.25, k, oi.ctypes.data_as(ctypes.c_void_p),
                                                od.ctypes.data_as(ctypes.c_void_p),
                                                osc.ctypes.data_as(ctypes.c_void_p)))
        t.append(time.perf_counter() - t0)
    out["c_call_prealloc_ms"] = round(1e3 * float(np.median(t)), 3)
    # device search + its own host-side enqueue cost, timed on the host
    t = []
    for _ in range(args.reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        idx.search_device(q.data_ptr(), nq, 64, 0.25, k, ids.data_ptr(), dists.data_ptr(), None, st)
        torch.cuda.synchronize()
        t.append(time.perf_counter() - t0)
    out["device_search_wall_ms"] = round(1e3 * float(np.median(t)), 3)
    # the same on the engine's private stream (stream NULL at the C ABI)
    t = []
    for _ in range(args.reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        _lib.check(_lib.lib().vlq_engine_search_device(idx._h, ctypes.c_void_p(q.data_ptr()), nq, 64, 0.25, k,
                                                       ctypes.c_void_p(ids.data_ptr()),
                                                       ctypes.c_void_p(dists.data_ptr()), None, None))
        idx.sync(None)
        t.append(time.perf_counter() - t0)
    out["device_search_engine_stream_wall_ms"] = round(1e3 * float(np.median(t)), 3)
    # traffic of one call alone
    pin_q = torch.empty((nq, w["dim"]), dtype=torch.float32).pin_memory()
    pin_i = torch.empty((nq, k), dtype=torch.int64).pin_memory()
    pin_d = torch.empty((nq, k), dtype=torch.float32).pin_memory()
    t = []
    for _ in range(args.reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        q.copy_(pin_q, non_blocking=True)
        pin_i.copy_(ids, non_blocking=True)
        pin_d.copy_(dists, non_blocking=True)
        torch.cuda.synchronize()
        t.append(time.perf_counter() - t0)
    out["pinned_copies_ms"] = round(1e3 * float(np.median(t)), 3)
    t = []
    for _ in range(args.reps):
        t0 = time.perf_counter()
        a = np.empty((nq, k), np.int64)
        b = np.empty((nq, k), np.float32)
        a[...] = pin_i.numpy()
        b[...] = pin_d.numpy()
        pin_q.numpy()[...] = qh
        t.append(time.perf_counter() - t0)
    out["host_memcpy_fresh_outputs_ms"] = round(1e3 * float(np.median(t)), 3)
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
