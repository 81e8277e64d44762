"""Generates tests/golden/* from the REFERENCE implementation itself.

Runs in the build container only (needs oracle/_ref, built from
/root/reference/proj by oracle/Makefile).  Every expected output below is
produced by the reference's own code:

* ``oracle/_ref/vlqadc`` -- the reference pybind11 module (bindings.cpp):
  Index.train / add / search / save, gen_synthetic, brute_force_gt;
* ``oracle/_ref/ref_tools`` -- acceptance make_instance replay
  (proj/tests/acceptance.cpp:74-115) and search_batch with SearchStats.

Fixtures (small; committed):
  <name>.model.vlq   trained quantizers, zero points (no t3)
  <name>.index.vlq   reference-built index (t3 stored, as Index.save writes it)
  <name>.npz         queries, base-generation params, expected search outputs
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

# (name, base params, query params, train params, search grid)
PY_CASES = [
    # the reference pytest smoke fixture (tests/python/test_smoke.py:10-21)
    ("smoke", dict(count=5000, dim=16, clusters=20, spread=0.05, seed=42),
     dict(count=50, dim=16, clusters=20, spread=0.05, seed=43),
     dict(k=32, n=8, m=4, iters=8, seed=1, clamp_lambda=True),
     [(16, 0.5, 10), (8, 0.5, 5), (32, 1.0, 10), (4, 0.25, 1), (2, 0.1, 100)]),
    # unclamped lambda range (index.cpp:110-132)
    ("unclamped", dict(count=4000, dim=8, clusters=12, spread=0.05, seed=7),
     dict(count=40, dim=8, clusters=12, spread=0.05, seed=8),
     dict(k=16, n=4, m=2, iters=6, seed=3, clamp_lambda=False),
     [(4, 0.5, 10), (16, 1.0, 20), (8, 0.25, 5)]),
    # m = 16 byte codes, D = 32 (DEEP-style 16-byte codes at toy scale)
    ("m16", dict(count=6000, dim=32, clusters=30, spread=0.05, seed=11),
     dict(count=40, dim=32, clusters=30, spread=0.05, seed=12),
     dict(k=64, n=8, m=16, iters=5, seed=5, clamp_lambda=True),
     [(16, 0.25, 100), (64, 1.0, 10), (8, 0.5, 32)]),
    # m = 8, D = 24, n = 1 (single edge per region)
    ("n1m8", dict(count=3000, dim=24, clusters=10, spread=0.1, seed=21),
     dict(count=30, dim=24, clusters=10, spread=0.1, seed=22),
     dict(k=20, n=1, m=8, iters=5, seed=9, clamp_lambda=True),
     [(5, 1.0, 10), (20, 1.0, 50), (3, 0.5, 7)]),
    # m = 1 (one sub-quantizer over the whole 4-D vector), tiny K
    ("m1", dict(count=1200, dim=4, clusters=6, spread=0.2, seed=31),
     dict(count=25, dim=4, clusters=6, spread=0.2, seed=32),
     dict(k=8, n=3, m=1, iters=5, seed=2, clamp_lambda=True),
     [(8, 1.0, 10), (2, 0.5, 3), (4, 0.3, 1000)]),
]

# acceptance "small" instance (acceptance.cpp:484-485), replayed by ref_tools
TOOL_CASES = [
    ("accept_small", [20000, 16, 40, 64, 8, 4, 8, 20000, 100, 1000, 0.05],
     [(16, 0.5, 10), (64, 1.0, 10), (8, 0.25, 100)]),
]


def ref_search_stats(index_path, queries_path, w1, alpha, k, tmp):
    out = os.path.join(tmp, "s.bin")
    subprocess.run([TOOLS, "search", index_path, queries_path, str(w1), repr(float(alpha)), str(k), out], check=True)
    return vlq1.read_ref_search(out)


def main():
    os.makedirs(HERE, exist_ok=True)
    with tempfile.TemporaryDirectory() as tmp:
        for name, bp, qp, tp, grid in PY_CASES:
            base = ref.gen_synthetic(bp["count"], bp["dim"], clusters=bp["clusters"], spread=bp["spread"],
                                     seed=bp["seed"])
            queries = ref.gen_synthetic(qp["count"], qp["dim"], clusters=qp["clusters"], spread=qp["spread"],
                                        seed=qp["seed"])
            idx = ref.Index.train(base, **tp)
            model_path = os.path.join(HERE, f"{name}.model.vlq")
            idx.save(model_path)
            # strip t3 from the model file to keep fixtures small (the reader
            # recomputes it: index_io.cpp:141-146)
            mdl = vlq1.read(model_path)
            vlq1.write(mdl, model_path, store_t3=False)
            idx.add(base)
            index_path = os.path.join(HERE, f"{name}.index.vlq")
            idx.save(index_path)  # reference Index.save: t3 stored
            qpath = os.path.join(tmp, "q.fvecs")
            vlq1.write_fvecs(queries, qpath)
            res = {}
            for gi, (w1, alpha, k) in enumerate(grid):
                ids, dists = idx.search(queries, w1=w1, alpha=alpha, k=k)
                rid, rd, scanned = ref_search_stats(index_path, qpath, w1, alpha, k, tmp)
                assert np.array_equal(rid, ids) and np.array_equal(rd.view(np.uint32), dists.view(np.uint32))
                res[f"ids_{gi}"] = ids
                res[f"dists_{gi}"] = dists
                res[f"scanned_{gi}"] = np.uint64(scanned)
            gt = ref.brute_force_gt(base, queries, 10)
            np.savez_compressed(os.path.join(HERE, f"{name}.npz"), queries=queries,
                                grid=np.array(grid, dtype=np.float64),
                                base_params=np.array([bp["count"], bp["dim"], bp["clusters"], bp["spread"],
                                                      bp["seed"]], np.float64),
                                gt10=gt, base_head=base[:64], **res)
            print(name, os.path.getsize(index_path), "bytes")
        for name, args, grid in TOOL_CASES:
            prefix = os.path.join(tmp, name)
            subprocess.run([TOOLS, "instance", *map(str, args), prefix], check=True)
            ix = vlq1.read(prefix + ".vlq")
            index_path = os.path.join(HERE, f"{name}.index.vlq")
            vlq1.write(ix, index_path, store_t3=False)
            queries = vlq1.read_fvecs(prefix + ".queries.fvecs")
            res = {}
            for gi, (w1, alpha, k) in enumerate(grid):
                rid, rd, scanned = ref_search_stats(prefix + ".vlq", prefix + ".queries.fvecs", w1, alpha, k, tmp)
                res[f"ids_{gi}"] = rid
                res[f"dists_{gi}"] = rd
                res[f"scanned_{gi}"] = np.uint64(scanned)
            base = vlq1.read_fvecs(prefix + ".base.fvecs")
            count, dim, clusters, spread, seed = args[0], args[1], args[2], args[10], args[9]
            np.savez_compressed(os.path.join(HERE, f"{name}.npz"), queries=queries,
                                grid=np.array(grid, dtype=np.float64),
                                base_params=np.array([count, dim, clusters, spread, seed], np.float64),
                                base_head=base[:64], **res)
            print(name, os.path.getsize(index_path), "bytes")


if __name__ == "__main__":
    main()
