#!/usr/bin/env python
"""VLQ-ADC batched search benchmark (BASELINE.json metric: QPS at fixed
recall@100 on synthetic data, B200 vs the reference CPU implementation).

A "step" is one batched search of the workload's full query batch (nq = 10k)
through the engine: coarse distances, first/second level selection, term5,
fused list scan + top-k', exact re-score.  Setup (untimed): GPU training of
the model on a prefix sample, streamed GPU add of the synthetic base, exact
GPU ground truth for a query subset.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--workload c2] [--impl ours|reference]

Under torchrun (N > 1) each rank holds the posting lists c with
shard_of_cell(c, N) == rank of the same index; each rank runs the first level
and the cell selection for 1/N of the batch, the selections (cells + exact
(a, b) pairs) are all-gathered (NCCL), every rank scans its shard for the
whole batch, and the per-shard exact top-k are all-gathered and merged by
(dist, id) (dist.ShardedIndex.search_select_split) -- scaling "strong" (the
index and batch are fixed, the lists are split).

`value` is device-timed (CUDA events, queries resident in HBM, L2 flushed
between steps, max over ranks).  `e2e` is the same metric through the public
API with host buffers (Index.search on numpy arrays: H2D of the queries and
D2H of ids/dists/scanned inside the timed region).  `cpu_baseline` times the
REFERENCE implementation (oracle/_ref, built from /root/reference/proj)
searching the same index (exported as VLQ1) on a bounded query sample.
"""
from __future__ import annotations

import argparse
import datetime
import json
import os
import statistics
import subprocess
import sys
import tempfile
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))


def w2_of(w1: int, alpha: float, n: int) -> int:
    """QueryParams::w2 (search.hpp:16-20)."""
    full = w1 * n
    w = int(float(np.float32(alpha)) * full)
    return min(max(w, 1), full)
sys.path.insert(0, ROOT)

METRIC = "QPS at fixed recall@100, 1B×96 synthetic, 1/2/4/8 B200 vs CPU ref"

# BASELINE.json configs; SURVEY.md §8d parameters (sigma = 0.05, base seed 42,
# query seed 43, n = 32 edges, w1 = 64, alpha = 0.25, k = 100)
WORKLOADS = {
    "tiny": dict(desc="tiny smoke workload: 200k x 32, K=256 x 16 lines, PQ 8 B", n=200_000, dim=32, k=256,
                 edges=16, m=8, clusters=256, ntrain=50_000),
    "c1": dict(desc="SIFT1M-shaped synthetic (configs[0]): 1M x 128, K=1024 x 32 lines, PQ 8 B, nq=10k, k=100",
               n=1_000_000, dim=128, k=1024, edges=32, m=8, clusters=1000, ntrain=100_000),
    "c2": dict(desc="DEEP10M-shaped synthetic (configs[1]): 10M x 96, K=4096 x 32 lines, PQ 16 B, nq=10k, k=100",
               n=10_000_000, dim=96, k=4096, edges=32, m=16, clusters=4000, ntrain=200_000),
    "deep100m": dict(desc="DEEP100M-shaped synthetic (HBM-resident scan study): 100M x 96, K=4096 x 32 lines, PQ 16 B, "
                          "nq=10k, k=100", n=100_000_000, dim=96, k=4096, edges=32, m=16, clusters=4000,
                     ntrain=200_000),
    "c4s": dict(desc="C4 coarse-stage study: 50M x 96, K=65536 x 32 lines, PQ 16 B, nq=10k, k=100 (C4's model "
                     "shape on a 1/20 base)", n=50_000_000, dim=96, k=65536, edges=32, m=16, clusters=65536,
                ntrain=2_000_000, gt_queries=1000),
    "c3": dict(desc="SIFT100M-shaped synthetic (configs[2]): 100M x 128, K=65536 x 32 lines, PQ 8 B, nq=10k, k=100",
               n=100_000_000, dim=128, k=65536, edges=32, m=8, clusters=65536, ntrain=2_000_000, gt_queries=1000),
    "c4": dict(desc="DEEP1B-shaped synthetic (configs[3]): 1B x 96, K=65536 x 32 lines, PQ 16 B, nq=10k, k=100",
               n=1_000_000_000, dim=96, k=65536, edges=32, m=16, clusters=65536, ntrain=2_000_000, gt_queries=1000),
    "c5": dict(desc="SIFT1B-shaped synthetic (configs[4]): 1B x 128, K=65536 x 32 lines, PQ 8 B, k=100",
               n=1_000_000_000, dim=128, k=65536, edges=32, m=8, clusters=65536, ntrain=2_000_000, gt_queries=1000),
}
SPREAD, BASE_SEED, QUERY_SEED, TRAIN_SEED = 0.05, 42, 43, 1


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def measured_peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return {}


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.rows = []
        self.proc = None

    def __enter__(self):
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap,utilization.gpu")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 8:
                self.rows.append(parts)

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        busy = [r for r in self.rows if r[7].isdigit() and int(r[7]) > 0] or self.rows
        sm = [float(r[0]) for r in busy if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in busy for i in range(4) if r[3 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows), "samples_under_load": len(busy)}


def build_index(vlqadc, w, device, rank=0, world=1):
    """Untimed setup: GPU training on a prefix sample (rank 0; the model is
    broadcast to the other ranks), streamed GPU add of each rank's shard."""
    import torch
    import torch.distributed as dist
    # scripts/shard_probe.py builds one rank's shard alone (no process group): it trains itself
    collective = world > 1 and dist.is_initialized()
    t0 = time.time()
    model = None
    if rank == 0 or not collective:
        sample = torch.empty((w["ntrain"], w["dim"]), dtype=torch.float32, device=f"cuda:{device}")
        vlqadc.gen_synthetic_device(0, w["ntrain"], w["dim"], w["clusters"], SPREAD, BASE_SEED, sample.data_ptr(),
                                    device=device)
        torch.cuda.synchronize(device)
        trained = vlqadc.Index.train(sample.cpu().numpy(), k=w["k"], n=w["edges"], m=w["m"], iters=10,
                                     seed=TRAIN_SEED, device=device)
        model = trained.model()
        del trained, sample
    if collective:
        box = [model]
        dist.broadcast_object_list(box, src=0)
        model = box[0]
    digest = model_digest(model)
    if collective:
        digests = [None] * world
        dist.all_gather_object(digests, digest)
        assert len(set(digests)) == 1, f"ranks hold different models: {digests}"
    idx = vlqadc.Index.from_model(model["dim"], model["k"], model["n"], model["m"], model["clamp"], model["lo"],
                                  model["hi"], model["centroids"], model["nbr"], model["elen"], model["pq"],
                                  device=device, shard_rank=rank, shard_count=world)
    t1 = time.time()
    idx.add_synthetic(w["n"], clusters=w["clusters"], spread=SPREAD, seed=BASE_SEED)
    t2 = time.time()
    log(f"[setup] rank {rank}: train {t1 - t0:.1f}s, add {w['n']} points {t2 - t1:.1f}s, "
        f"local entries {idx.local_entries}, model {digest}")
    return idx, {"train_s": round(t1 - t0, 2), "add_s": round(t2 - t1, 2), "train_points": w["ntrain"],
                 "model_sha256_16": digest}


def model_digest(model) -> str:
    import hashlib
    h = hashlib.sha256()
    for key in ("centroids", "nbr", "elen", "pq"):
        h.update(np.ascontiguousarray(model[key]).tobytes())
    h.update(np.array([model["lo"], model["hi"]], np.float32).tobytes())
    return h.hexdigest()[:16]


def make_queries(vlqadc, w, nq, device, kind="ref"):
    """kind "ref": the reference's convention (README.md:79-80, acceptance.cpp:113):
    gen_synthetic with another seed, i.e. another set of cluster centres, so
    the queries lie outside the base mixture.  kind "heldout": fresh rows
    n, n+1, ... of the base generator -- the same mixture as the base (how
    DEEP1B / SIFT1B queries relate to their bases)."""
    import torch
    q = torch.empty((nq, w["dim"]), dtype=torch.float32, device=f"cuda:{device}")
    first, seed = (w["n"], BASE_SEED) if kind == "heldout" else (0, QUERY_SEED)
    vlqadc.gen_synthetic_device(first, nq, w["dim"], w["clusters"], SPREAD, seed, q.data_ptr(), device=device)
    torch.cuda.synchronize(device)
    return q


def recall_at(ids: np.ndarray, gt: np.ndarray, k: int) -> float:
    """recall_at (proj/src/eval.cpp:13-36): true NN = gt column 0 in the first k ids."""
    hit = (ids[:, :k] == gt[:, :1].astype(np.int64)).any(axis=1)
    return float(hit.mean())


def ref_module():
    ref = os.path.join(ROOT, "oracle", "_ref")
    if not os.path.isdir(os.path.join(ref, "vlqadc")):
        raise RuntimeError("oracle/_ref not built (run __graft_entry__.build() where /root/reference exists)")
    if ref not in sys.path:
        sys.path.insert(0, ref)
    import vlqadc as refmod  # the reference's own pybind11 module
    return refmod


def time_reference(ref_idx, refmod, queries: np.ndarray, w1, alpha, k, budget_s: float, warm: int = 100):
    """Reference Index.search on a bounded sample with all host threads
    (set_max_threads(0) = hardware_concurrency, parallel.cpp:17-24)."""
    refmod.set_max_threads(0)
    cores = os.cpu_count() or 1
    ref_idx.search(queries[:warm], w1=w1, alpha=alpha, k=k)  # warm-up excluded (eval.cpp:91)
    probe = queries[warm:warm + 200]
    t = time.perf_counter()
    ref_idx.search(probe, w1=w1, alpha=alpha, k=k)
    rate1 = len(probe) / max(time.perf_counter() - t, 1e-6)  # serial: parallel_for runs < 1024 queries on one thread
    # >= 256 queries per host thread so parallel_for (parallel.cpp:27-40) occupies every core
    ns = int(min(len(queries) - warm, max(256 * cores, rate1 * cores * budget_s)))
    sample = queries[warm:warm + ns]
    t = time.perf_counter()
    ids, dists = ref_idx.search(sample, w1=w1, alpha=alpha, k=k)
    dt = time.perf_counter() - t
    return ns / dt, ns, dt, ids, dists, warm


def time_port(idx, queries: np.ndarray, w1, alpha, k, budget_s: float, warm: int = 100):
    """The C restatement of the reference search (oracle/, test infrastructure)
    on host copies of the GPU-built index: for 1e8-1e9-point indexes where a
    VLQ1 round trip through the reference is tens of GB of file I/O."""
    from oracle import oracle as orc, vlq1
    mdl = idx.model()
    off, ids, codes, lams = idx.lists()
    ix = vlq1.Vlq1(mdl["dim"], mdl["k"], mdl["n"], mdl["m"], mdl["clamp"], mdl["lo"], mdl["hi"], mdl["centroids"],
                   mdl["nbr"], mdl["elen"], mdl["pq"], None, off, ids, codes, lams)
    o = orc.OracleIndex(ix)
    o.search(queries[:warm], w1, alpha, k)
    probe = queries[warm:warm + 50]
    t = time.perf_counter()
    o.search(probe, w1, alpha, k)
    rate = len(probe) / max(time.perf_counter() - t, 1e-6)
    ns = int(min(len(queries) - warm, max(50, rate * budget_s)))
    sample = queries[warm:warm + ns]
    t = time.perf_counter()
    rids, rd, _ = o.search(sample, w1, alpha, k)
    dt = time.perf_counter() - t
    return ns / dt, ns, dt, rids, rd, warm


def add_replay(vlqadc, idx, w, npoints: int, device: int, seed: int = 7, full_cells: int = 24) -> dict:
    """Sampled add-path parity of a built index (proj/tests/test_index.cpp:161-189
    pattern) without copying the index to the host.  The base generator is
    counter-based, so any row i is regenerated on the device.
      1. `npoints` rows (blocks of 1000 consecutive ids at seeded random
         starts): the GPU encode (Index.encode) and the oracle's assign on host
         copies of the model give the same (cell, exact lambda, code, lambda
         byte) bit for bit;
      2. each sampled id is present in the STORED list of its oracle cell with
         that code and lambda byte, and every fetched list is ascending by id;
      3. `full_cells` whole stored lists: every entry's row, regenerated and
         assigned by the oracle, maps to that cell with the stored code and
         lambda byte (no foreign entries)."""
    import torch
    from oracle import oracle as orc, vlq1  # the checker
    t0 = time.time()
    mdl = idx.model()
    o = orc.OracleIndex(vlq1.Vlq1(mdl["dim"], mdl["k"], mdl["n"], mdl["m"], mdl["clamp"], mdl["lo"], mdl["hi"],
                                  mdl["centroids"], mdl["nbr"], mdl["elen"], mdl["pq"]))
    rng = np.random.default_rng(seed)
    blk = 1000
    nblk = max(1, npoints // blk)
    starts = np.sort(rng.choice(max(1, (w["n"] - blk) // blk), size=nblk, replace=False)) * blk
    buf = torch.empty((nblk * blk, w["dim"]), dtype=torch.float32, device=f"cuda:{device}")
    for b, s0 in enumerate(starts):
        vlqadc.gen_synthetic_device(int(s0), blk, w["dim"], w["clusters"], SPREAD, BASE_SEED,
                                    buf[b * blk].data_ptr(), device=device)
    torch.cuda.synchronize(device)
    x = buf.cpu().numpy()
    rows = (starts[:, None] + np.arange(blk)[None, :]).ravel().astype(np.int64)
    gc, gl, gcd, glb = idx.encode(x)
    oc, ol, ocd, olb = o.assign(x)
    encode_ok = bool(np.array_equal(gc, oc) and np.array_equal(gl.view(np.uint32), ol.view(np.uint32)) and
                     np.array_equal(gcd, ocd) and np.array_equal(glb, olb))
    # 2. presence in the stored lists
    ucells, inv = np.unique(oc, return_inverse=True)
    counts, ids, codes, lams = idx.cells(ucells)
    seg = np.zeros(len(ucells) + 1, np.int64)
    np.cumsum(counts.astype(np.int64), out=seg[1:])
    sorted_ok = all(bool(np.all(np.diff(ids[seg[i]:seg[i + 1]].astype(np.int64)) > 0)) for i in range(len(ucells)))
    present = 0
    for p_ in range(len(rows)):
        a, b = seg[inv[p_]], seg[inv[p_] + 1]
        j = a + int(np.searchsorted(ids[a:b], rows[p_]))
        if j < b and ids[j] == rows[p_] and np.array_equal(codes[j], ocd[p_]) and lams[j] == olb[p_]:
            present += 1
    # 3. whole lists: no foreign entries
    nonempty = np.flatnonzero(counts > 0)
    pick = rng.choice(nonempty, size=min(full_cells, len(nonempty)), replace=False)
    ent_ids = np.concatenate([ids[seg[i]:seg[i + 1]] for i in pick])
    ent_cell = np.concatenate([np.full(int(counts[i]), ucells[i], np.uint32) for i in pick])
    ent_codes = np.concatenate([codes[seg[i]:seg[i + 1]] for i in pick])
    ent_lams = np.concatenate([lams[seg[i]:seg[i + 1]] for i in pick])
    xr = torch.empty((len(ent_ids), w["dim"]), dtype=torch.float32, device=f"cuda:{device}")
    for r, i in enumerate(ent_ids):
        vlqadc.gen_synthetic_device(int(i), 1, w["dim"], w["clusters"], SPREAD, BASE_SEED, xr[r].data_ptr(),
                                    device=device)
    torch.cuda.synchronize(device)
    fc, _, fcd, flb = o.assign(xr.cpu().numpy())
    lists_ok = bool(np.array_equal(fc, ent_cell) and np.array_equal(fcd, ent_codes) and np.array_equal(flb, ent_lams))
    return {"add_replay_bit_exact": bool(encode_ok and present == len(rows) and sorted_ok and lists_ok),
            "points": int(len(rows)), "encode_bit_exact_vs_oracle": encode_ok,
            "present_in_stored_list": int(present), "lists_ascending": bool(sorted_ok),
            "whole_lists_checked": int(len(pick)), "whole_list_entries": int(len(ent_ids)),
            "whole_lists_bit_exact": lists_ok, "seconds": round(time.time() - t0, 1),
            "method": "rows regenerated by the counter-based generator; oracle assign (oracle/vlq_oracle.c) on "
                      "host copies of the model vs Index.encode and vs the stored posting lists (vlq_engine_get_cells)"}


def config_of(args, w, world):
    return {"workload": w["desc"], "n_base": w["n"], "dim": w["dim"], "K": w["k"], "n_edges": w["edges"],
            "m_bytes": w["m"], "nq": args.nq, "w1": args.w1, "alpha": args.alpha, "k": args.k,
            "train_points": w["ntrain"],
            "parallelism": f"list-sharded x{world} (hashed cells)" if world > 1 else "single GPU",
            "l2": "flushed between steps (512 MiB write)", "data": "synthetic Gaussian mixture (sigma 0.05)"}


def self_launch(n: int) -> int:
    """`bench.py --gpus N` outside torchrun: one process per GPU under
    torch.distributed.run on 127.0.0.1 (the driver's own launch line)."""
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__), *sys.argv[1:]]
    log(f"[launch] {' '.join(cmd)}")
    return subprocess.call(cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--workload", default="c4", choices=sorted(WORKLOADS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--nq", type=int, default=10_000)
    ap.add_argument("--w1", type=int, default=64)
    ap.add_argument("--alpha", type=float, default=0.25)
    ap.add_argument("--k", type=int, default=100)
    ap.add_argument("--gt-queries", type=int, default=None, help="queries with exact ground truth (default per workload)")
    ap.add_argument("--cpu-kind", default=None, choices=["reference", "port"],
                    help="CPU baseline: the reference via a VLQ1 file (default up to 1e8 points) or the C oracle port")
    ap.add_argument("--cpu-budget", type=float, default=12.0, help="seconds of reference CPU work per sample")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--sweep", default=None,
                    help="comma-separated w1 values: device QPS and recall@1/10/100 per w1 (QPS-recall curve)")
    ap.add_argument("--ivf", action="store_true",
                    help="also build and time the IVFADC comparison baseline (ivf_baseline.cpp) on the same model, w = w1")
    ap.add_argument("--profile", action="store_true",
                    help="wrap the timed steps in cudaProfilerStart/Stop (for ncu --profile-from-start off) and exit")
    ap.add_argument("--replay-points", type=int, default=100_000,
                    help="sampled base rows whose add-path outputs are replayed against the oracle")
    ap.add_argument("--ref-setup", default=None, help=argparse.SUPPRESS)  # internal: reference-arm index builder
    args = ap.parse_args()
    args.warmup = max(3, args.warmup)

    multi = os.environ.get("VLQ_MULTI", "group")  # group: one process drives N GPUs; procs: one process per GPU
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ and (multi == "procs" or args.impl == "reference"):
        # one process per GPU: re-launch this command under torch.distributed.run
        sys.exit(self_launch(args.gpus))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if world > 1 and world != args.gpus:
        raise SystemExit(f"bench: --gpus {args.gpus} but WORLD_SIZE={world}")
    if args.ref_setup:
        ref_setup(args)
        return
    if args.impl == "reference":
        run_reference_arm(args, rank, world)
        return
    if args.gpus > 1 and multi == "group":
        run_group(args, rank, world)
        return

    import torch
    import torch.distributed as dist

    # one process per GPU; VLQ_DIST_BACKEND=gloo (with ranks sharing GPUs
    # round-robin) is the single-GPU rehearsal of the N > 1 path
    local = int(os.environ.get("LOCAL_RANK", "0")) % max(1, torch.cuda.device_count())
    backend = os.environ.get("VLQ_DIST_BACKEND", "nccl")
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
        else:
            dist.init_process_group(backend)
    torch.cuda.set_device(local)
    os.environ["VLQ_DEVICE"] = str(local)
    w = WORKLOADS[args.workload]
    cfg = config_of(args, w, world)

    from paper_1901_00275_b200 import vlqadc
    from paper_1901_00275_b200.dist import ShardedIndex

    idx, setup = build_index(vlqadc, w, local, rank, world)
    q = make_queries(vlqadc, w, args.nq, local)
    nq, k = args.nq, args.k
    ids = torch.empty((nq, k), dtype=torch.int64, device=q.device)
    dists = torch.empty((nq, k), dtype=torch.float32, device=q.device)
    scanned = torch.empty((nq,), dtype=torch.int64, device=q.device)
    flush = torch.empty(512 << 20, dtype=torch.uint8, device=q.device)
    # one dedicated stream for the L2 flush, the events and every engine /
    # NCCL launch, so the flush is ordered before each timed step
    stream = torch.cuda.Stream(q.device)
    torch.cuda.set_stream(stream)
    st = stream.cuda_stream

    sharded = ShardedIndex(idx) if world > 1 else None

    def step():
        if sharded is not None:  # query-split coarse stage + selection, sharded scan, K9 merge
            mi, md, _ = sharded.search_select_split(q, args.w1, args.alpha, k, out=(ids, dists, scanned))
            return mi, md
        idx.search_device(q.data_ptr(), nq, args.w1, args.alpha, k, ids.data_ptr(), dists.data_ptr(),
                          scanned.data_ptr(), st)
        return ids, dists

    for _ in range(args.warmup):
        step()
    idx.sync(st)
    torch.cuda.synchronize()
    # per-phase CUDA events ride along on the same stream (no host sync until
    # stats() after the timed region)
    idx.set_profiling(True)
    idx.stats(reset=True)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    if args.profile:
        torch.cuda.profiler.start()
    with ClockSampler(local) as clocks:
        for s in range(args.steps):
            flush.zero_()
            ev[s][0].record(stream)
            out_ids, out_d = step()
            ev[s][1].record(stream)
        torch.cuda.synchronize()
    if args.profile:
        torch.cuda.profiler.stop()
        log(f"[profile] {args.steps} steps, {sum(a.elapsed_time(b) for a, b in ev):.3f} ms (under profiler: not a bench value)")
        return
    if world > 1:
        dist.barrier()
    idx.sync(st)
    ms = sum(a.elapsed_time(b) for a, b in ev)
    stats = idx.stats()
    idx.set_profiling(False)
    red_dev = q.device if backend == "nccl" else "cpu"  # gloo reduces host tensors
    t_max = torch.tensor([ms], dtype=torch.float64, device=red_dev)
    if world > 1:
        dist.all_reduce(t_max, op=dist.ReduceOp.MAX)
    ms_max = float(t_max.item())
    value = nq * args.steps / (ms_max / 1e3)

    # algorithmic bytes of the dominant kernel (the fused list scan): S_q*(m+5)
    local_scanned = int(scanned.sum().item())
    scan_bytes_per_step = local_scanned * (w["m"] + 5)
    scan_ms = stats["phase_ms"]["scan"] / args.steps
    res_ids = out_ids.cpu().numpy()
    res_d = out_d.cpu().numpy()

    e2e = None
    if world > 1:
        # every rank copies the batch in (pinned), runs the query-split search;
        # rank 0 reads the merged result back; device time, max over ranks
        qpin = torch.from_numpy(q.cpu().numpy()).pin_memory()
        qdev = torch.empty_like(q)
        e_ms = 0.0
        for s_ in range(args.steps + 1):
            dist.barrier()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            qdev.copy_(qpin, non_blocking=True)
            mi, md, _ = sharded.search_select_split(qdev, args.w1, args.alpha, k, out=(ids, dists, scanned))
            if rank == 0:
                e_ids = mi.to("cpu", non_blocking=True)
                e_d = md.to("cpu", non_blocking=True)
            e1.record(stream)
            torch.cuda.synchronize()
            if s_ > 0:  # the first call is a warm-up
                e_ms += e0.elapsed_time(e1)
        t_e = torch.tensor([e_ms], dtype=torch.float64, device=red_dev)
        dist.all_reduce(t_e, op=dist.ReduceOp.MAX)
        e2e = {"value": round(nq * args.steps / (float(t_e.item()) / 1e3), 1), "unit": "queries/s",
               "h2d_bytes_per_step": int(qpin.numel() * 4), "d2h_bytes_per_step": int(nq * k * 12),
               "api": "ShardedIndex.search_select_split (pinned host queries in, merged ids/dists out on rank 0)",
               "timing": "CUDA events around H2D + search + D2H, max over ranks"}

    if rank != 0:
        dist.barrier()
        dist.destroy_process_group()
        return

    peaks = measured_peaks()
    hbm = float(peaks.get("hbm_gbs", 6650.0))
    # workload shape: scanned entries per query (S_q) and list lengths
    sq = scanned.cpu().numpy().astype(np.float64)
    lens = np.diff(idx.list_offsets().astype(np.int64))
    reg = lens.reshape(w["k"], w["edges"]).sum(axis=1)
    shape = {"scanned_per_query": {"mean": round(float(sq.mean()), 1), "p50": float(np.percentile(sq, 50)),
                                   "p99": float(np.percentile(sq, 99)), "max": float(sq.max())},
             "uniform_model_scanned_per_query": round(w2_of(args.w1, args.alpha, w["edges"]) * w["n"] /
                                                      (w["k"] * w["edges"]), 1),
             "list_len": {"mean": round(float(lens.mean()), 2), "p99": float(np.percentile(lens, 99)),
                          "max": int(lens.max()), "empty_frac": round(float((lens == 0).mean()), 4)},
             "region_len": {"mean": round(float(reg.mean()), 2), "p99": float(np.percentile(reg, 99)),
                            "max": int(reg.max())}}
    # the coarse contraction (first_level_scan's nq x K x D distances) on the
    # tensor cores: logical 2 nq K D FLOP against the dense TF32 rate; the
    # "coarse" phase is the relayout of the query rows + the one tcgen05 pass
    coarse_ms = stats["phase_ms"]["coarse"] / args.steps
    gemm_flop = 2.0 * nq * w["k"] * w["dim"]
    bf16 = peaks.get("bf16_tflops")
    tf32_peak = float(bf16) / 2.0 if bf16 else 1100.0
    gemm = {"bound": "tensor", "kernel": "k_coarse_tc<4> (tcgen05.mma kind::tf32, 1xTF32, TMEM accumulators, "
                                         "8-centroid chunk-minimum epilogue)",
            "flop_per_launch": gemm_flop, "coarse_ms_per_step": round(coarse_ms, 4),
            "achieved": round(gemm_flop / (coarse_ms / 1e3) / 1e12, 1) if coarse_ms > 0 else None,
            "peak": round(tf32_peak, 1), "unit": "TFLOP/s",
            "peak_source": ("MEASURED_PEAKS.json bf16_tflops / 2 (the dense TF32 rate is half the bf16 rate)"
                            if bf16 else "fallback: 1.1 PFLOP/s dense TF32 (datasheet)"),
            "tc_used": bool(w["k"] >= 16384 and w["dim"] % 8 == 0)}
    if coarse_ms > 0:
        gemm["frac"] = round(gemm["achieved"] / tf32_peak, 4)
    achieved = scan_bytes_per_step / (scan_ms / 1e3) / 1e9 if scan_ms > 0 else None
    traffic = None
    tr_path = os.path.join(ROOT, "profiles", f"scan_traffic_{args.workload}.json")
    if os.path.exists(tr_path):
        traffic = json.load(open(tr_path)).get("dram_bytes_per_launch")
    roofline = {"bound": "hbm", "kernel": "k_scan<M,fast> (fused list scan + warp top-k')",
                "achieved": round(achieved, 1) if achieved else None, "peak": hbm, "unit": "GB/s",
                "frac": round(achieved / hbm, 4) if achieved else None, "traffic": traffic,
                "peak_source": "MEASURED_PEAKS.json hbm_gbs (measured copy)" if peaks else "fallback 6650",
                "algorithmic_bytes_per_launch": scan_bytes_per_step,
                "bytes_per_candidate": w["m"] + 5, "scan_ms_per_launch": round(scan_ms, 4),
                "phase_ms_per_step": {p: round(v / args.steps, 4) for p, v in stats["phase_ms"].items()},
                "scan_share_of_step": round(scan_ms / (ms_max / args.steps), 4), "gemm": gemm}

    # recall on the exact ground truth of a query subset
    ngt = min(args.gt_queries or w.get("gt_queries", 1000), nq)
    qh = q.cpu().numpy()
    gt = vlqadc.brute_force_gt_synthetic(w["n"], w["dim"], w["clusters"], SPREAD, BASE_SEED, qh[:ngt], 1,
                                         device=local)
    recall = {f"recall@{r}": round(recall_at(res_ids[:ngt], gt, r), 4) for r in (1, 10, 100) if r <= k}
    # the same search on held-out queries of the base mixture (not timed)
    qho = make_queries(vlqadc, w, ngt, local, kind="heldout").cpu().numpy()
    gt_ho = vlqadc.brute_force_gt_synthetic(w["n"], w["dim"], w["clusters"], SPREAD, BASE_SEED, qho, 1, device=local)
    if world == 1:
        ho_ids, _ = idx.search(qho, w1=args.w1, alpha=args.alpha, k=k)
        recall["heldout"] = {f"recall@{r}": round(recall_at(ho_ids, gt_ho, r), 4) for r in (1, 10, 100) if r <= k}
        recall["heldout"]["queries"] = (f"{ngt} fresh rows of the base generator (same mixture); the main figures "
                                        f"use the reference's query convention (another seed = other centres)")

    # e2e: public API with host buffers (H2D queries + D2H results per step)
    if world == 1:
        import gc
        for _ in range(args.warmup):  # the same W warm-up calls as the device-timed steps
            idx.search(qh, w1=args.w1, alpha=args.alpha, k=k)
        per = []
        gc.collect()
        gc.disable()  # no collector pause inside a timed call (the outputs are fresh numpy arrays)
        try:
            for _ in range(args.steps):
                t = time.perf_counter()
                e_ids, e_d = idx.search(qh, w1=args.w1, alpha=args.alpha, k=k)
                per.append(time.perf_counter() - t)
        finally:
            gc.enable()
        e2e_s = sum(per)
        assert np.array_equal(e_ids, res_ids)
        e2e = {"value": round(nq * args.steps / e2e_s, 1), "unit": "queries/s",
               "h2d_bytes_per_step": int(qh.nbytes), "d2h_bytes_per_step": int(nq * k * 12 + nq * 8),
               "api": "paper_1901_00275_b200.vlqadc.Index.search (numpy in/out)",
               "ms_per_call": [round(1e3 * x, 2) for x in per]}

    cpu = None
    parity = None
    if world == 1 and not args.no_cpu_baseline:
        kind = args.cpu_kind or ("reference" if w["n"] <= 100_000_000 else "port")
        try:
            if kind == "reference":
                refmod = ref_module()
                with tempfile.TemporaryDirectory() as tmp:
                    path = os.path.join(tmp, "bench.vlq")
                    idx.save(path)
                    ref_idx = refmod.Index.load(path)
                qps, ns, dt, rids, rd, off = time_reference(ref_idx, refmod, qh, args.w1, np.float32(args.alpha), k,
                                                            args.cpu_budget)
                del ref_idx
                what = "reference Index.search (oracle/_ref) on the same index via VLQ1, set_max_threads(0)"
            else:
                qps, ns, dt, rids, rd, off = time_port(idx, qh, args.w1, np.float32(args.alpha), k, args.cpu_budget)
                what = "C oracle port (oracle/vlq_oracle.c) on host copies of the same index, all host threads"
            parity = bool(np.array_equal(rids, res_ids[off:off + ns]) and
                          np.array_equal(rd.view(np.uint32), res_d[off:off + ns].view(np.uint32)))
            cpu = {"value": round(qps, 2), "unit": "queries/s", "cores": os.cpu_count(), "kind": kind,
                   "sample": f"{ns} of the {nq} benchmark queries (after 100 warm-up), {what}, {dt:.1f} s",
                   "ids_and_dists_bit_exact_vs_gpu": parity}
        except Exception as e:  # reported, never silently replaced
            cpu = {"value": None, "kind": kind, "unavailable": f"{type(e).__name__}: {e}"}

    replay = None
    if world == 1 and args.replay_points > 0:
        try:
            replay = add_replay(vlqadc, idx, w, args.replay_points, local)
        except Exception as e:  # reported, never silently replaced
            replay = {"add_replay_bit_exact": None, "unavailable": f"{type(e).__name__}: {e}"}
        log(f"[replay] {replay}")

    sweep = None
    if args.sweep and world == 1:
        sweep = []
        for sw1 in [int(x) for x in args.sweep.split(",") if x]:
            for _ in range(2):
                idx.search_device(q.data_ptr(), nq, sw1, args.alpha, k, ids.data_ptr(), dists.data_ptr(),
                                  scanned.data_ptr(), st)
            torch.cuda.synchronize()
            sms = 0.0
            for _ in range(max(3, args.steps // 2)):
                flush.zero_()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                idx.search_device(q.data_ptr(), nq, sw1, args.alpha, k, ids.data_ptr(), dists.data_ptr(),
                                  scanned.data_ptr(), st)
                e1.record(stream)
                torch.cuda.synchronize()
                sms += e0.elapsed_time(e1)
            reps = max(3, args.steps // 2)
            sids = ids.cpu().numpy()
            sweep.append({"w1": sw1, "alpha": args.alpha, "qps": round(nq * reps / (sms / 1e3), 1),
                          "ms_per_step": round(sms / reps, 3),
                          "scanned_per_query": round(float(scanned.sum().item()) / nq, 1),
                          **{f"recall@{r}": round(recall_at(sids[:ngt], gt, r), 4) for r in (1, 10, 100) if r <= k}})
            log(f"[sweep] {sweep[-1]}")

    ivf_line = None
    if args.ivf and world == 1:
        t0 = time.time()
        ivf = vlqadc.build_ivf_baseline_synthetic(w["n"], idx, clusters=w["clusters"], spread=SPREAD, seed=BASE_SEED)
        build_s = time.time() - t0
        for _ in range(args.warmup):
            ivf.search_device(q.data_ptr(), nq, args.w1, k, ids.data_ptr(), dists.data_ptr(), scanned.data_ptr(), st)
        torch.cuda.synchronize()
        ivf_ms = 0.0
        for _ in range(args.steps):
            flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            ivf.search_device(q.data_ptr(), nq, args.w1, k, ids.data_ptr(), dists.data_ptr(), scanned.data_ptr(), st)
            e1.record(stream)
            torch.cuda.synchronize()
            ivf_ms += e0.elapsed_time(e1)
        iv_ids = ids.cpu().numpy()
        ivf_line = {"system": "ivfadc (ivf_baseline.cpp, exact GPU port)", "w": args.w1,
                    "value": round(nq * args.steps / (ivf_ms / 1e3), 1), "unit": "queries/s",
                    "ms_per_step": round(ivf_ms / args.steps, 3),
                    "scanned_per_query": round(float(scanned.sum().item()) / nq, 1), "build_s": round(build_s, 1),
                    "recall": {f"recall@{r}": round(recall_at(iv_ids[:ngt], gt, r), 4) for r in (1, 10, 100)
                               if r <= k}}

    clk = clocks.summary()
    line = {"metric": METRIC, "value": round(value, 1), "unit": "queries/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(ms_max / args.steps, 4), "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f32 (exact reference order) + u8 codes",
            "data": "synthetic", "config": cfg, "recall": recall, "e2e": e2e, "roofline": roofline,
            "cpu_baseline": cpu, "gpu_launches": stats["launches"] + (args.steps if world > 1 else 0),
            "coarse_stage": ("query-split first level + cell selection (1/N of the batch per rank), "
                             "selections all-gathered") if world > 1 else "single GPU",
            "ivfadc": ivf_line, "sweep": sweep, "add_replay": replay, "workload_shape": shape,
            "clocks": clk, "setup": setup, "scanned_per_query": round(local_scanned / nq, 1) if world == 1 else None,
            "fallback_queries_per_step": stats["flagged"] / args.steps,
            "tc_coarse_fallbacks_per_step": stats["tc_fallbacks"] / args.steps}
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def run_group(args, rank, world):
    """N > 1: the index sharded over N GPUs of this box behind ONE process
    (vlqadc.IndexGroup = the C-ABI vlq_group, csrc/group.cu): engine g on GPU g
    holds the lists c with shard_of_cell(c, N) == g; each step runs the
    query-split selection, the sharded scan reading the selections over NVLink
    peer memory and the per-slice merge of the shards' top-k from peer memory.
    Under torchrun (the driver's launch) rank 0 drives all N GPUs and the other
    ranks only wait; the step time is the device time of the batch, max over
    the GPUs (CUDA events on every GPU's stream)."""
    import torch
    import torch.distributed as dist
    N = args.gpus
    if world > 1:
        # the other ranks wait out rank 0's whole run (1B-point adds included)
        dist.init_process_group("gloo", timeout=datetime.timedelta(hours=3))
        if rank != 0:
            dist.barrier()  # rank 0 has finished
            dist.destroy_process_group()
            return
    # VLQ_GROUP_DEVICES="0,0": the single-GPU rehearsal (N shard engines on one GPU)
    devices = [int(x) for x in os.environ.get("VLQ_GROUP_DEVICES", ",".join(map(str, range(N)))).split(",")]
    if len(devices) != N:
        raise SystemExit(f"bench: --gpus {N} but VLQ_GROUP_DEVICES lists {len(devices)} devices")
    if torch.cuda.device_count() <= max(devices):
        raise SystemExit(f"bench: --gpus {N} but {torch.cuda.device_count()} visible GPUs")
    udev = sorted(set(devices))
    # S-way list sharding x N/S replicas (each replica searches 1/(N/S) of the
    # batch): 2-way list sharding, N/2 replicas of it.  Measured member by
    # member at C4 (profiles/r2_shard_probe_c4_final2.jsonl),
    # N = 8: S = 2 x R = 4 projects 6.6x, S = 4 x R = 2 6.0x, S = 8 5.3x --
    # the per-GPU work that does not shrink with the shard (selection, term5,
    # re-score, the scan's per-query prologue) is done for fewer queries
    S = int(os.environ.get("VLQ_GROUP_SHARDS", str(min(N, 2))))
    from paper_1901_00275_b200 import vlqadc
    w = WORKLOADS[args.workload]
    cfg = config_of(args, w, N)
    cfg["parallelism"] = (f"list-sharded x{S} (hashed cells) x {N // S} replica(s), one process driving {N} GPUs "
                          f"(vlq_group, NVLink P2P)")
    if os.environ.get("VLQ_GROUP_DEVICES"):
        cfg["parallelism"] += f"; rehearsal on devices {os.environ['VLQ_GROUP_DEVICES']}"
    t0 = time.time()
    sample = torch.empty((w["ntrain"], w["dim"]), dtype=torch.float32, device="cuda:0")
    vlqadc.gen_synthetic_device(0, w["ntrain"], w["dim"], w["clusters"], SPREAD, BASE_SEED, sample.data_ptr(), device=0)
    torch.cuda.synchronize(0)
    trained = vlqadc.Index.train(sample.cpu().numpy(), k=w["k"], n=w["edges"], m=w["m"], iters=10, seed=TRAIN_SEED,
                                 device=0)
    model = trained.model()
    del trained, sample
    t1 = time.time()
    grp = vlqadc.IndexGroup.from_model(model, devices, shards=S)
    grp.add_synthetic(w["n"], clusters=w["clusters"], spread=SPREAD, seed=BASE_SEED)
    t2 = time.time()
    local = grp.local_entries()
    log(f"[setup] group of {N}: train {t1 - t0:.1f}s, add {w['n']} points {t2 - t1:.1f}s, shards {local}")
    setup = {"train_s": round(t1 - t0, 2), "add_s": round(t2 - t1, 2), "train_points": w["ntrain"],
             "model_sha256_16": model_digest(model), "shard_entries": local}
    qh = make_queries(vlqadc, w, args.nq, 0).cpu().numpy()
    nq, k = args.nq, args.k
    flush = [torch.empty(512 << 20, dtype=torch.uint8, device=f"cuda:{g}") for g in udev]
    grp.set_queries(qh)
    for _ in range(args.warmup):
        grp.search_resident(args.w1, args.alpha, k)
    grp.set_profiling(True)
    for g in range(N):
        grp.stats(g, reset=True)
    ms_steps = []
    with ClockSampler(0) as clocks:
        for _ in range(args.steps):
            for f in flush:
                f.zero_()
            for g in udev:
                torch.cuda.synchronize(g)
            ms_steps.append(grp.search_resident(args.w1, args.alpha, k))
    stats = [grp.stats(g) for g in range(N)]
    grp.set_profiling(False)
    ms = sum(ms_steps)
    value = nq * args.steps / (ms / 1e3)
    res_ids, res_d, scanned = grp.results()
    # e2e through the public API: host queries in, merged host results out
    for _ in range(args.warmup):
        grp.search(qh, w1=args.w1, alpha=args.alpha, k=k)
    per = []
    for _ in range(args.steps):
        t = time.perf_counter()
        e_ids, e_d = grp.search(qh, w1=args.w1, alpha=args.alpha, k=k)
        per.append(time.perf_counter() - t)
    assert np.array_equal(e_ids, res_ids)
    e2e = {"value": round(nq * args.steps / sum(per), 1), "unit": "queries/s", "h2d_bytes_per_step": int(qh.nbytes * N),
           "d2h_bytes_per_step": int(nq * k * 12), "api": "paper_1901_00275_b200.vlqadc.IndexGroup.search (numpy in/out)",
           "ms_per_call": [round(1e3 * x, 2) for x in per]}
    peaks = measured_peaks()
    hbm = float(peaks.get("hbm_gbs", 6650.0))
    scan_bytes = int(scanned.sum()) * (w["m"] + 5)
    scan_ms = [st["phase_ms"]["scan"] / args.steps for st in stats]
    # per GPU: its share of the algorithmic bytes over its own scan time; the
    # line reports the slowest GPU's rate (the one that sets the step)
    # member g: shard g % S of replica g / S, which searches 1/R of the batch
    shard_bytes = [scan_bytes * local[g] / max(1, sum(local)) for g in range(N)]
    rates = [shard_bytes[g] / (scan_ms[g] / 1e3) / 1e9 if scan_ms[g] > 0 else 0.0 for g in range(N)]
    gslow = int(np.argmax(scan_ms))
    roofline = {"bound": "hbm", "kernel": "k_scan_fast2 (fused list scan + top-k'), per GPU",
                "achieved": round(rates[gslow], 1), "peak": hbm, "unit": "GB/s",
                "frac": round(rates[gslow] / hbm, 4) if rates[gslow] else None, "traffic": None,
                "per_gpu_achieved": [round(r, 1) for r in rates],
                "per_gpu_scan_ms": [round(x, 4) for x in scan_ms],
                "algorithmic_bytes_per_step": scan_bytes,
                "note": "shard bytes estimated as the batch's algorithmic bytes x the shard's share of the entries",
                "phase_ms_per_step_gpu0": {p: round(v / args.steps, 4) for p, v in stats[0]["phase_ms"].items()},
                "peak_source": "MEASURED_PEAKS.json hbm_gbs (measured copy)" if peaks else "fallback 6650"}
    ngt = min(args.gt_queries or w.get("gt_queries", 1000), nq)
    gt = vlqadc.brute_force_gt_synthetic(w["n"], w["dim"], w["clusters"], SPREAD, BASE_SEED, qh[:ngt], 1, device=0)
    recall = {f"recall@{r}": round(recall_at(res_ids[:ngt], gt, r), 4) for r in (1, 10, 100) if r <= k}
    line = {"metric": METRIC, "value": round(value, 1), "unit": "queries/s", "n_gpus": N, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(ms / args.steps, 4), "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f32 (exact reference order) + u8 codes",
            "data": "synthetic", "config": cfg, "recall": recall, "e2e": e2e, "roofline": roofline,
            "cpu_baseline": None, "gpu_launches": sum(st["launches"] for st in stats) + 2 * N * args.steps,
            "timing": "CUDA events on every GPU's stream around each batch, max over the GPUs; L2 flushed on every GPU",
            "clocks": clocks.summary(), "setup": setup, "scanned_per_query": round(float(scanned.sum()) / nq, 1),
            "fallback_queries_per_step": sum(st["flagged"] for st in stats) / args.steps}
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def ref_setup(args):
    """Child process of the reference arm: builds the workload's index on the
    GPU (the reference needs hours to train / add at these sizes),
    exports it as VLQ1 and writes the queries plus the GPU's own results, so
    the timed reference process never maps libvlqgpu.so."""
    import torch
    from paper_1901_00275_b200 import vlqadc
    out = args.ref_setup
    w = WORKLOADS[args.workload]
    idx, setup = build_index(vlqadc, w, 0)
    q = make_queries(vlqadc, w, args.nq, 0)
    ids = torch.empty((args.nq, args.k), dtype=torch.int64, device=q.device)
    dists = torch.empty((args.nq, args.k), dtype=torch.float32, device=q.device)
    scanned = torch.empty((args.nq,), dtype=torch.int64, device=q.device)
    idx.search_device(q.data_ptr(), args.nq, args.w1, args.alpha, args.k, ids.data_ptr(), dists.data_ptr(),
                      scanned.data_ptr(), 0)
    idx.sync(0)
    np.save(os.path.join(out, "queries.npy"), q.cpu().numpy())
    np.save(os.path.join(out, "gpu_ids.npy"), ids.cpu().numpy())
    np.save(os.path.join(out, "gpu_dists.npy"), dists.cpu().numpy())
    t0 = time.time()
    idx.save(os.path.join(out, "bench.vlq"))
    setup["vlq1_save_s"] = round(time.time() - t0, 1)
    json.dump(setup, open(os.path.join(out, "setup.json"), "w"))


def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def run_reference_arm(args, rank, world):
    """--impl reference: the reference's own CPU search (oracle/_ref, its
    unmodified sources compiled by oracle/Makefile) on the same workload, on
    the box's host cores.  The index is built on the GPU in a child process
    (ref_setup) and handed over as a VLQ1 file; this process loads only the
    reference module.  Timed: Index.search on bounded query slices with
    set_max_threads(0) (hardware_concurrency, parallel.cpp:17-24), plus a
    set_max_threads(1) sample; every searched slice is checked bit-exact
    against the GPU's results for the same queries.  Under torchrun only rank
    0 runs."""
    if rank != 0:
        return
    w = WORKLOADS[args.workload]
    cfg = config_of(args, w, 1)
    refmod = ref_module()
    with tempfile.TemporaryDirectory(dir=os.environ.get("VLQ_REF_TMP")) as tmp:
        env = {k: v for k, v in os.environ.items()
               if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "LOCAL_WORLD_SIZE", "MASTER_ADDR", "MASTER_PORT",
                            "GROUP_RANK", "ROLE_RANK", "TORCHELASTIC_RUN_ID")}
        t0 = time.time()
        subprocess.run([sys.executable, os.path.abspath(__file__), "--ref-setup", tmp, "--workload", args.workload,
                        "--nq", str(args.nq), "--w1", str(args.w1), "--alpha", str(args.alpha), "--k", str(args.k)],
                       env=env, check=True)
        t1 = time.time()
        path = os.path.join(tmp, "bench.vlq")
        gb = os.path.getsize(path) / 1e9
        ref_idx = refmod.Index.load(path)
        log(f"[reference] GPU build + VLQ1 export {t1 - t0:.1f}s ({gb:.1f} GB), reference load {time.time() - t1:.1f}s")
        qh = np.load(os.path.join(tmp, "queries.npy"))
        gids = np.load(os.path.join(tmp, "gpu_ids.npy"))
        gd = np.load(os.path.join(tmp, "gpu_dists.npy"))
        setup = json.load(open(os.path.join(tmp, "setup.json")))
    alpha = np.float32(args.alpha)
    parity = {"queries_checked": 0, "mismatched_queries": 0}

    def search(lo, hi):
        ids, d = ref_idx.search(qh[lo:hi], w1=args.w1, alpha=alpha, k=args.k)
        bad = ~((ids == gids[lo:hi]).all(axis=1) & (d.view(np.uint32) == gd[lo:hi].view(np.uint32)).all(axis=1))
        parity["queries_checked"] += hi - lo
        parity["mismatched_queries"] += int(bad.sum())

    refmod.set_max_threads(0)
    cores = os.cpu_count() or 1
    search(0, 100)  # warm-up excluded (eval.cpp:91)
    t = time.perf_counter()
    search(100, 300)
    rate1 = 200 / max(time.perf_counter() - t, 1e-6)  # < 1024 queries: parallel_for runs them serially
    # parallel_for (parallel.cpp:27-40) runs batches under 1024 queries on ONE
    # thread and cuts larger ones into chunks of >= 256 queries: a step needs
    # >= 256 x threads queries to occupy every host core
    per_step = int(min(args.nq - 300, max(256 * cores, rate1 * cores * 3.0)))
    times = []
    for s in range(args.warmup + args.steps):
        lo = 300 + (s * per_step) % max(1, args.nq - 300 - per_step)
        t = time.perf_counter()
        search(lo, lo + per_step)
        if s >= args.warmup:
            times.append(time.perf_counter() - t)
    value = per_step * len(times) / sum(times)
    # one host thread (set_max_threads(1)): a bounded sample of ~10 s
    refmod.set_max_threads(1)
    n1 = int(max(5, min(2000, 10.0 * rate1)))
    t = time.perf_counter()
    search(0, n1)
    one_thread = n1 / (time.perf_counter() - t)
    refmod.set_max_threads(0)
    sample = (f"{per_step} of the {args.nq} benchmark queries per step (slices after 300 warm-up/probe queries), "
              f"reference Index.search (oracle/_ref, unmodified sources), set_max_threads(0) = {cores} threads")
    line = {"impl": "reference", "metric": METRIC, "value": round(value, 2), "unit": "queries/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(1e3 * sum(times) / len(times), 2),
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": dict(cfg, reference_sample=f"{per_step} queries per step"),
            "cpu_baseline": {"value": round(value, 2), "unit": "queries/s", "cores": cores, "kind": "reference",
                             "cpu_model": cpu_model(), "sample": sample,
                             "one_thread": {"value": round(one_thread, 3), "unit": "queries/s", "queries": n1,
                                            "threads": 1}},
            "parity_vs_gpu": dict(parity, bit_exact=parity["mismatched_queries"] == 0,
                                  what="reference ids and distances vs the GPU engine's for the same queries"),
            "setup": setup,
            "e2e": {"value": round(value, 2), "unit": "queries/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
