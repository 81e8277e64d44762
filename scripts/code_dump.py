#!/usr/bin/env python
"""Dumps the PQ codes of a sample of posting lists of a built workload index
(GPU box) for offline bank-conflict studies of the scan's LUT lookups.

  python scripts/code_dump.py --workload c4 --cells 400 --out gpurun_out/codes_c4.npz
"""
import argparse
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="c4", choices=sorted(bench.WORKLOADS))
    ap.add_argument("--cells", type=int, default=400)
    ap.add_argument("--out", required=True)
    args = ap.parse_args()
    from paper_1901_00275_b200 import vlqadc
    w = bench.WORKLOADS[args.workload]
    idx, _ = bench.build_index(vlqadc, w, 0)
    off = idx.list_offsets().astype(np.int64)
    lens = np.diff(off)
    rng = np.random.default_rng(0)
    # cells weighted by length (the scan's work is per entry)
    p = lens / lens.sum()
    cells = np.unique(rng.choice(len(lens), size=args.cells, p=p)).astype(np.uint32)
    counts, ids, codes, lams = idx.cells(cells)
    np.savez_compressed(args.out, cells=cells, counts=counts, ids=ids, codes=codes, lams=lams)
    print("cells", len(cells), "entries", len(ids))


if __name__ == "__main__":
    main()
