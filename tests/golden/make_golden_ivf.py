"""Generates tests/golden/ivf_<name>.npz from the REFERENCE IVFADC baseline
(proj/src/ivf_baseline.cpp) via oracle/_ref/ref_tools (build container only).

For each case the reference builds the baseline index from the fixture's
model (codebook + PQ, as eval.cpp:182 does) and base set, and searches the
fixture's queries for a grid of (w, k).  Stored: the lists (list_off, ids,
codes) and the reference's ids / dists / scanned totals.
"""
from __future__ import annotations

import os
import subprocess
import sys
import tempfile

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
REF = os.path.join(ROOT, "oracle", "_ref")
sys.path.insert(0, REF)
import vlqadc as ref  # noqa: E402  (the reference's own module)

sys.path.insert(0, ROOT)
from oracle import vlq1  # noqa: E402

TOOLS = os.path.join(REF, "ref_tools")

# (fixture, model file, search grid of (w, k))
CASES = [
    ("smoke", "smoke.model.vlq", [(4, 10), (32, 10), (1, 5), (8, 100)]),
    ("m16", "m16.model.vlq", [(8, 100), (64, 10), (3, 32)]),
    ("n1m8", "n1m8.model.vlq", [(5, 10), (20, 50)]),
    ("m1", "m1.model.vlq", [(8, 10), (2, 1000)]),
    ("accept_small", "accept_small.index.vlq", [(16, 10), (64, 100), (4, 1)]),
]


def main():
    with tempfile.TemporaryDirectory() as tmp:
        for name, model, grid in CASES:
            z = dict(np.load(os.path.join(HERE, f"{name}.npz")))
            count, dim, clusters, spread, seed = z["base_params"]
            base = ref.gen_synthetic(int(count), int(dim), clusters=int(clusters), spread=float(spread),
                                     seed=int(seed))
            assert np.array_equal(base[:64], z["base_head"])
            bpath, qpath, out = (os.path.join(tmp, x) for x in ("b.fvecs", "q.fvecs", "ivf.bin"))
            vlq1.write_fvecs(base, bpath)
            vlq1.write_fvecs(z["queries"], qpath)
            res = {}
            lists = None
            for gi, (w, k) in enumerate(grid):
                subprocess.run([TOOLS, "ivf", os.path.join(HERE, model), bpath, qpath, str(w), str(k), out],
                               check=True)
                lists, (rid, rd, scanned) = vlq1.read_ref_ivf(out)
                res[f"ids_{gi}"] = rid
                res[f"dists_{gi}"] = rd
                res[f"scanned_{gi}"] = np.uint64(scanned)
            np.savez_compressed(os.path.join(HERE, f"ivf_{name}.npz"), grid=np.array(grid, np.int64),
                                list_off=lists[0], ids=lists[1], codes=lists[2], **res)
            print(name, "ivf lists", int(lists[0][-1]))


if __name__ == "__main__":
    main()
