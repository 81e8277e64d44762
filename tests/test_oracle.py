"""CPU tests: the oracle restatement is pinned against the reference's golden
vectors (tests/golden, produced by the reference itself) and the reference's
own known-answer tests.  No GPU needed."""
import os
import struct

import numpy as np
import pytest

from conftest import ALL_CASES, PY_CASES, grid_of, load_golden, regen_base
from oracle import oracle, vlq1


@pytest.mark.parametrize("name", ALL_CASES)
def test_oracle_search_matches_reference_golden(name):
    z, index_path, _ = load_golden(name)
    o = oracle.OracleIndex.load(index_path)
    for gi, (w1, alpha, k) in enumerate(grid_of(z)):
        ids, dists, scanned = o.search(z["queries"], w1, alpha, k)
        assert np.array_equal(ids, z[f"ids_{gi}"]), (name, gi)
        assert np.array_equal(dists.view(np.uint32), z[f"dists_{gi}"].view(np.uint32)), (name, gi)
        assert int(scanned.sum()) == int(z[f"scanned_{gi}"]), (name, gi)


@pytest.mark.parametrize("name", PY_CASES + ["accept_small"])
def test_oracle_build_matches_reference_lists(name):
    z, index_path, model_path = load_golden(name)
    want = vlq1.read(index_path)
    model = vlq1.read(model_path) if model_path else vlq1.Vlq1(
        want.dim, want.k, want.n, want.m, want.clamp, want.lo, want.hi, want.centroids, want.nbr, want.elen, want.pq)
    if model_path is None:
        model.lo, model.hi = 0.0, 1.0
    base = regen_base(z)
    got = oracle.OracleIndex(model).build(base)
    assert (np.float32(got.lo), np.float32(got.hi)) == (np.float32(want.lo), np.float32(want.hi))
    assert np.array_equal(got.list_off, want.list_off)
    assert np.array_equal(got.ids, want.ids)
    assert np.array_equal(got.codes, want.codes)
    assert np.array_equal(got.lambdas, want.lambdas)


@pytest.mark.parametrize("name", PY_CASES)
def test_vlq1_roundtrip_is_byte_identical(name, tmp_path):
    _, index_path, _ = load_golden(name)
    ix = vlq1.read(index_path)
    out = str(tmp_path / "rt.vlq")
    vlq1.write(ix, out, store_t3=True)
    assert open(out, "rb").read() == open(index_path, "rb").read()
    assert os.path.getsize(index_path) == vlq1.expected_size(ix.dim, ix.k, ix.n, ix.m, ix.ntotal, True)


@pytest.mark.parametrize("name", PY_CASES)
def test_oracle_t3_equals_reference_t3(name):
    _, index_path, _ = load_golden(name)
    ix = vlq1.read(index_path)  # t3 written by the reference (compute_t3)
    t3 = oracle.compute_t3(ix.centroids, ix.pq)
    assert np.array_equal(t3.view(np.uint32), ix.t3.view(np.uint32))


def test_vlq1_errors(tmp_path):
    _, index_path, _ = load_golden("smoke")
    raw = open(index_path, "rb").read()
    bad = tmp_path / "bad.vlq"
    bad.write_bytes(b"XXXX" + raw[4:])
    with pytest.raises(RuntimeError, match="bad magic"):
        vlq1.read(str(bad))
    bad.write_bytes(raw[: len(raw) // 2])
    with pytest.raises(RuntimeError, match="truncated"):
        vlq1.read(str(bad))
    bad.write_bytes(raw[:4] + struct.pack("<I", 2) + raw[8:])
    with pytest.raises(RuntimeError, match="unsupported version"):
        vlq1.read(str(bad))


# ---- known-answer tests from the reference suites ---------------------------

def test_lambda_quantizer_kats():
    # proj/tests/test_index.cpp:44-69
    q = oracle.quantize_lambda
    assert q(0.0, 0.0, 1.0) == 0 and q(1.0, 0.0, 1.0) == 255
    assert q(-0.3, 0.0, 1.0) == 0 and q(1.7, 0.0, 1.0) == 255
    assert q(-2.0, -2.0, 3.0) == 0 and q(3.0, -2.0, 3.0) == 255
    assert oracle.dequantize_lambda(0, 0.0, 1.0) == np.float32(0.5 / 256)
    assert oracle.dequantize_lambda(255, 0.0, 1.0) == np.float32(1.0 - 0.5 / 256)
    rng = np.random.default_rng(30)
    lo, hi = np.float32(-0.25), np.float32(1.25)
    bound = (hi - lo) / 512 + 1e-9
    for lam in rng.uniform(lo, hi, 2000).astype(np.float32):
        back = oracle.dequantize_lambda(q(float(lam), float(lo), float(hi)), float(lo), float(hi))
        assert abs(back - lam) <= bound


def test_line_quantization_kats():
    # proj/tests/test_quantizers.cpp:194-205
    assert oracle.line_lambda(0.0, 4.0, 4.0) == 0.0
    assert oracle.line_lambda(4.0, 0.0, 4.0) == 1.0
    assert oracle.line_lambda(2.0, 2.0, 4.0) == 0.5
    assert abs(oracle.line_sqdist(1.0, 1.0, 4.0, 0.5)) < 1e-6
    assert abs(oracle.line_sqdist(2.0, 2.0, 4.0, 0.5) - 1.0) < 1e-6


def test_compute_t3_hand_case():
    # proj/tests/test_index.cpp:71-86: <(1,2), (3,4)> = 11
    cent = np.array([[1, 2, 0, 0]], np.float32)
    pq = np.zeros((2, 256, 2), np.float32)
    pq[0, 0] = [3, 4]
    t3 = oracle.compute_t3(cent, pq)
    assert t3[0, 0, 0] == 11.0


def test_w2_formula():
    # QueryParams::w2 (search.hpp:16-20)
    assert oracle.w2(64, 0.25, 32) == 512
    assert oracle.w2(1, 0.01, 4) == 1
    assert oracle.w2(4, 1.0, 4) == 16
    assert oracle.w2(3, 2.0, 5) == 15


def test_adc_decomposition_matches_direct_evaluation():
    # proj/tests/test_search.cpp:198-224 / acceptance C1 (rel 1e-4)
    z, index_path, _ = load_golden("smoke")
    o = oracle.OracleIndex.load(index_path)
    ix = o.ix
    for y in z["queries"][:5]:
        ws, t5 = o.query_tables(y)
        ynorm = float(np.dot(y, y))
        for cell in range(0, ix.k * ix.n, 7):
            i, j = divmod(cell, ix.n)
            for e in range(int(ix.list_off[cell]), int(ix.list_off[cell + 1])):
                got = o.adc_distance(ws, t5, ix.codes[e], int(ix.lambdas[e]), i, j)
                want = o.direct_adc(y, ix.codes[e], int(ix.lambdas[e]), i, j)
                assert abs(got - want) <= 1e-4 * max(1e-3, abs(want), ynorm)


IVF_CASES = ["smoke", "m16", "n1m8", "m1", "accept_small"]


def _ivf_fixture(name):
    from conftest import GOLDEN
    z = dict(np.load(os.path.join(GOLDEN, f"ivf_{name}.npz")))
    model = os.path.join(GOLDEN, f"{name}.model.vlq")
    if not os.path.exists(model):
        model = os.path.join(GOLDEN, f"{name}.index.vlq")
    return z, model


@pytest.mark.parametrize("name", IVF_CASES)
def test_oracle_ivf_baseline_matches_reference_golden(name):
    """The C restatement of build_ivf_baseline / search_ivf_baseline
    (ivf_baseline.cpp) reproduces the reference's lists and results
    bit-exactly (fixtures made by the reference itself,
    tests/golden/make_golden_ivf.py)."""
    z, model = _ivf_fixture(name)
    g, _, _ = load_golden(name)
    o = oracle.OracleIndex(vlq1.read(model))
    base = regen_base(g)
    off, ids, codes = o.ivf_build(base)
    assert np.array_equal(off, z["list_off"]) and np.array_equal(ids, z["ids"])
    assert np.array_equal(codes, z["codes"])
    for gi, (w, k) in enumerate(z["grid"]):
        rid, rd, sc = o.ivf_search((off, ids, codes), g["queries"], int(w), int(k))
        assert np.array_equal(rid, z[f"ids_{gi}"]), (name, gi)
        assert np.array_equal(rd.view(np.uint32), z[f"dists_{gi}"].view(np.uint32)), (name, gi)
        assert int(sc.sum()) == int(z[f"scanned_{gi}"])


def test_oracle_ivf_exhaustive_equals_full_adc():
    """test_eval.cpp "w=k is exhaustive-ADC-exact": w = K scans every list."""
    z, model = _ivf_fixture("smoke")
    g, _, _ = load_golden("smoke")
    o = oracle.OracleIndex(vlq1.read(model))
    base = regen_base(g)
    lists = o.ivf_build(base)
    rid, rd, sc = o.ivf_search(lists, g["queries"], o.ix.k, 10)
    assert (sc == len(base)).all()
    with pytest.raises(RuntimeError, match="search_ivf_baseline: need 0 < w <= k"):
        o.ivf_search(lists, g["queries"], 0, 10)


# Index.train arguments of the golden models (tests/golden/make_golden.py PY_CASES)
TRAIN_PARAMS = {"smoke": dict(k=32, iters=8, seed=1), "unclamped": dict(k=16, iters=6, seed=3),
                "m16": dict(k=64, iters=5, seed=5), "n1m8": dict(k=20, iters=5, seed=9),
                "m1": dict(k=8, iters=5, seed=2)}


@pytest.mark.parametrize("name", PY_CASES)
def test_oracle_train_kmeans_equals_reference_codebook(name, oracle_mod):
    """The k-means restatement (oracle/train_oracle.cpp) reproduces the
    reference's trained first-level codebook bit for bit: the golden models
    were written by the reference's Index.train, whose codebook is
    train_kmeans(train, k, iters, seed) (bindings.cpp:57)."""
    tp = TRAIN_PARAMS[name]
    z, _, model_path = load_golden(name)
    base = regen_base(z)
    mdl = vlq1.read(model_path)
    got = oracle_mod.train_kmeans(base, tp["k"], tp["iters"], tp["seed"])
    assert np.array_equal(got.view(np.uint32), mdl.centroids.view(np.uint32))
    # seeding + Lloyd from the seeds is the same computation
    seeds = oracle_mod.kmeans_seed(base, tp["k"], tp["seed"])
    again = oracle_mod.kmeans_lloyd(base, seeds, tp["iters"])
    assert np.array_equal(again.view(np.uint32), mdl.centroids.view(np.uint32))
