#!/usr/bin/env python
"""How much of a query's scan could a distance lower bound skip? (GPU box.)

Builds the workload's index (as bench.py), searches a few queries for their
final top-k' threshold tau (the k'-th exact distance), recomputes the second
level in numpy, and for every selected cell / entry evaluates
  cell  bound: (sqrt(min_lambda t1) - rmax_cell)^2
  entry bound: (sqrt(t1(lambda_e)) - |r^_e|)^2
(reverse triangle inequality, |r^_e|^2 = sum_p t2[p][code_p]).  Prints the
fractions of entries whose bound exceeds tau.
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
    ap.add_argument("--workload", default="c4")
    ap.add_argument("--nq", type=int, default=16)
    ap.add_argument("--w1", type=int, default=64)
    ap.add_argument("--alpha", type=float, default=0.25)
    ap.add_argument("--keep", type=int, default=128)
    args = ap.parse_args()
    from paper_1901_00275_b200 import vlqadc
    from oracle import oracle as orc
    w = bench.WORKLOADS[args.workload]
    idx, _ = bench.build_index(vlqadc, w, 0)
    q = bench.make_queries(vlqadc, w, 1000, 0).cpu().numpy()[: args.nq]
    ids, d = idx.search(q, w1=args.w1, alpha=args.alpha, k=args.keep)
    tau = d[:, -1]
    mdl = idx.model()
    off, _, codes, lams = idx.lists()
    C, nbr, elen, pq = mdl["centroids"], mdl["nbr"], mdl["elen"], mdl["pq"]
    n, m = mdl["n"], mdl["m"]
    t2 = orc.compute_t2(pq)
    lo, hi = idx.lambda_range
    delta = (hi - lo) / 256.0
    w2 = max(1, int(float(np.float32(args.alpha)) * args.w1 * n))
    out = []
    for qi in range(args.nq):
        y = q[qi].astype(np.float64)
        ws = ((C.astype(np.float64) - y) ** 2).sum(1)
        top = np.argsort(ws, kind="stable")[: args.w1]
        cells, ld = [], []
        for i in top:
            for j in range(n):
                a, b, c = ws[i], ws[nbr[i, j]], float(elen[i, j])
                lam = min(max(0.5 * (a + c - b) / c, 0.0), 1.0)
                ld.append((1 - lam) * a + (lam * lam - lam) * c + lam * b)
                cells.append(i * n + j)
        sel = np.array(cells)[np.argsort(np.array(ld), kind="stable")[:w2]]
        tot = cell_pr = ent_pr = 0
        for cell in sel:
            b0, b1 = int(off[cell]), int(off[cell + 1])
            if b0 == b1:
                continue
            i, j = cell // n, cell % n
            a, b, c = ws[i], ws[nbr[i, j]], float(elen[i, j])
            lam = lo + (lams[b0:b1].astype(np.float64) + 0.5) * delta
            t1 = a + lam * ((b - a - c) + lam * c)
            cd = codes[b0:b1].astype(np.int64)
            r = np.sqrt(t2[np.arange(m)[None, :], cd].sum(1))
            lbe = np.where(np.sqrt(np.maximum(t1, 0)) > r, (np.sqrt(np.maximum(t1, 0)) - r) ** 2, 0.0)
            lam_lo, lam_hi = lo + 0.5 * delta, lo + 255.5 * delta
            ls = min(max(-(b - a - c) / (2 * c), lam_lo), lam_hi)
            t1m = a + ls * ((b - a - c) + ls * c)
            lbc = (np.sqrt(max(t1m, 0)) - r.max()) ** 2 if np.sqrt(max(t1m, 0)) > r.max() else 0.0
            tot += b1 - b0
            cell_pr += (b1 - b0) if lbc > tau[qi] else 0
            ent_pr += int((lbe > tau[qi]).sum())
        out.append({"q": qi, "tau": float(tau[qi]), "entries": tot, "cell_prunable": cell_pr / max(tot, 1),
                    "entry_prunable": ent_pr / max(tot, 1)})
        print(json.dumps(out[-1]), flush=True)
    print(json.dumps({"mean_cell_prunable": float(np.mean([o["cell_prunable"] for o in out])),
                      "mean_entry_prunable": float(np.mean([o["entry_prunable"] for o in out]))}), flush=True)


if __name__ == "__main__":
    main()
