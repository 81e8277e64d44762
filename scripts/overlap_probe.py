#!/usr/bin/env python
"""How much scan work could two queries share?  (GPU box only.)

Builds the workload's index, runs the selection stage for the batch, then
measures, for every query, the scanned entries it shares with its best
partner (the query whose selected cells cover the most of its own entries)
and the fraction a greedy pairing of the whole batch would scan once instead
of twice.  Answers whether a paired (two queries per pass over a cell) scan
could cut the per-entry LSU work.

  python scripts/overlap_probe.py --workload c4
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
    ap.add_argument("--nq", type=int, default=10_000)
    ap.add_argument("--w1", type=int, default=64)
    ap.add_argument("--alpha", type=float, default=0.25)
    ap.add_argument("--heldout", action="store_true", help="queries from the base mixture")
    args = ap.parse_args()
    import torch
    from paper_1901_00275_b200 import vlqadc
    w = bench.WORKLOADS[args.workload]
    idx, setup = bench.build_index(vlqadc, w, 0)
    if args.heldout:
        q = torch.empty((args.nq, w["dim"]), dtype=torch.float32, device="cuda:0")
        vlqadc.gen_synthetic_device(w["n"], args.nq, w["dim"], w["clusters"], bench.SPREAD, bench.BASE_SEED,
                                    q.data_ptr(), device=0)
    else:
        q = bench.make_queries(vlqadc, w, args.nq, 0)
    nq = args.nq
    w2 = idx.w2(args.w1, args.alpha)
    sel = torch.empty((nq, w2), dtype=torch.int32, device="cuda:0")
    ab = torch.empty((nq, w2, 2), dtype=torch.float32, device="cuda:0")
    idx.search_select_device(q.data_ptr(), nq, args.w1, args.alpha, sel.data_ptr(), ab.data_ptr())
    torch.cuda.synchronize()
    off = torch.from_numpy(idx.list_offsets().astype(np.int64)).cuda()
    ncell = off.numel() - 1
    ln = (off[1:] - off[:-1]).double()
    cells = sel.long()
    lens = ln[cells]  # [nq, w2]
    per_q = lens.sum(1)
    # S[a, b] = entries of a's cells that b also scans = sum_c len(c) [c in a][c in b]
    rows = torch.arange(nq, device="cuda:0").repeat_interleave(w2)
    Aw = torch.sparse_coo_tensor(torch.stack([rows, cells.reshape(-1)]), lens.reshape(-1).float(),
                                 (nq, ncell)).coalesce()
    S = torch.empty((nq, nq), dtype=torch.float32, device="cuda:0")
    nb = 256
    for b0 in range(0, nq, nb):
        b1 = min(nq, b0 + nb)
        B = torch.zeros((ncell, b1 - b0), dtype=torch.float32, device="cuda:0")
        cols = torch.arange(b1 - b0, device="cuda:0").repeat_interleave(w2)
        B[cells[b0:b1].reshape(-1), cols] = 1.0
        S[:, b0:b1] = torch.sparse.mm(Aw, B)
        del B
    S.fill_diagonal_(0)
    best, partner = S.max(1)
    frac_best = (best.double() / per_q).cpu().numpy()
    # greedy pairing by shared entries (largest first)
    Sc = S.clone()
    order = torch.argsort(S.max(1).values, descending=True).cpu().numpy()
    used = np.zeros(nq, bool)
    shared = 0.0
    Sh = Sc.cpu().numpy()
    for a in order:
        if used[a]:
            continue
        row = Sh[a].copy()
        row[used] = -1
        row[a] = -1
        b = int(row.argmax())
        if row[b] <= 0:
            used[a] = True
            continue
        used[a] = used[b] = True
        shared += float(min(Sh[a, b], Sh[b, a]))
    total = float(per_q.sum().item())
    out = {"workload": args.workload, "queries": "heldout" if args.heldout else "reference convention", "nq": nq,
           "w2": w2, "entries_per_query": total / nq,
           "best_partner_shared_frac": {"mean": float(frac_best.mean()), "p50": float(np.median(frac_best)),
                                        "p90": float(np.percentile(frac_best, 90))},
           "greedy_pairing_entries_saved_frac": shared / total}
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
