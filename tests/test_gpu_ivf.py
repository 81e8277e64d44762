"""GPU IVFADC comparison baseline (csrc/ivf.cu) against the REFERENCE's own
build_ivf_baseline / search_ivf_baseline outputs (tests/golden/ivf_*.npz,
made by tests/golden/make_golden_ivf.py through oracle/_ref/ref_tools) and the
C oracle: lists, ids, distances and scanned counts bit-exact."""
import os

import numpy as np
import pytest

from conftest import GOLDEN, load_golden, regen_base

pytestmark = pytest.mark.gpu

IVF_CASES = ["smoke", "m16", "n1m8", "m1", "accept_small"]


def same_f32(a, b):
    return np.array_equal(np.asarray(a, np.float32).view(np.uint32), np.asarray(b, np.float32).view(np.uint32))


def _fixture(name):
    z = dict(np.load(os.path.join(GOLDEN, f"ivf_{name}.npz")))
    model = os.path.join(GOLDEN, f"{name}.model.vlq")
    if not os.path.exists(model):
        model = os.path.join(GOLDEN, f"{name}.index.vlq")
    g, _, _ = load_golden(name)
    return z, model, g


@pytest.fixture(params=["auto", "tc"])
def vlqadc(request, monkeypatch):
    import torch
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    if request.param == "tc":  # tensor-core assignment + coarse stage forced on
        monkeypatch.setenv("VLQ_TC_MIN_K", "0")
    from paper_1901_00275_b200 import vlqadc as mod
    return mod


@pytest.mark.parametrize("name", IVF_CASES)
def test_ivf_build_and_search_match_reference_golden(vlqadc, name):
    z, model, g = _fixture(name)
    idx = vlqadc.Index.load(model)
    base = regen_base(g)
    ivf = vlqadc.build_ivf_baseline(base, idx)
    assert ivf.base_count == len(base)
    off, ids, codes = ivf.lists()
    assert np.array_equal(off, z["list_off"]) and np.array_equal(ids, z["ids"])
    assert np.array_equal(codes, z["codes"])
    for gi, (w, k) in enumerate(z["grid"]):
        rid, rd, sc = vlqadc.search_ivf_baseline(ivf, g["queries"], int(w), int(k), return_scanned=True)
        assert np.array_equal(rid, z[f"ids_{gi}"]), (name, gi)
        assert same_f32(rd, z[f"dists_{gi}"]), (name, gi)
        assert int(sc.sum()) == int(z[f"scanned_{gi}"]), (name, gi)


def test_ivf_random_parameters_and_exhaustive_match_oracle(vlqadc, oracle_mod):
    """w = K is exhaustive (test_eval.cpp "w=k is exhaustive-ADC-exact") and
    random (w, k) agree with the C oracle over the same lists."""
    from oracle import vlq1
    rng = np.random.default_rng(3)
    for name in ("m16", "accept_small"):
        z, model, g = _fixture(name)
        idx = vlqadc.Index.load(model)
        base = regen_base(g)
        ivf = vlqadc.build_ivf_baseline(base, idx)
        o = oracle_mod.OracleIndex(vlq1.read(model))
        lists = ivf.lists()
        params = [(idx.k, 10), (idx.k, 100)] + [(int(rng.integers(1, idx.k + 1)), int(rng.choice([1, 7, 64, 300])))
                                               for _ in range(4)]
        for w, k in params:
            rid, rd, sc = vlqadc.search_ivf_baseline(ivf, g["queries"], w, k, return_scanned=True)
            oid, od, osc = o.ivf_search(lists, g["queries"], w, k)
            assert np.array_equal(rid, oid) and same_f32(rd, od), (name, w, k)
            assert np.array_equal(sc, osc)
        full = vlqadc.search_ivf_baseline(ivf, g["queries"], idx.k, 5, return_scanned=True)[2]
        assert (full == len(base)).all()


def test_ivf_centroid_base_gives_zero_residual_codes(vlqadc):
    """test_eval.cpp "base equal to the centroids gives near-zero residual
    codes": every list entry carries the code of the zero vector."""
    from oracle import vlq1
    _, model, _ = _fixture("smoke")
    mdl = vlq1.read(model)
    idx = vlqadc.Index.load(model)
    ivf = vlqadc.build_ivf_baseline(mdl.centroids, idx)
    off, ids, codes = ivf.lists()
    assert len(ids) == mdl.k
    zero_idx = vlqadc.Index.load(model)
    zc = vlqadc.build_ivf_baseline(np.zeros((1, mdl.dim), np.float32) + mdl.centroids[:1], zero_idx).lists()[2]
    assert (codes == zc[0]).all()


def test_ivf_errors_mirror_reference(vlqadc):
    z, model, g = _fixture("smoke")
    idx = vlqadc.Index.load(model)
    with pytest.raises(RuntimeError, match="no baseline index built"):
        vlqadc.search_ivf_baseline(vlqadc.IvfBaselineIndex(idx), g["queries"], 4, 10)
    with pytest.raises(RuntimeError, match="build_ivf_baseline: dimension mismatch"):
        vlqadc.build_ivf_baseline(np.zeros((3, idx.dim + 1), np.float32), idx)
    ivf = vlqadc.build_ivf_baseline(regen_base(g), idx)
    with pytest.raises(RuntimeError, match="search_ivf_baseline: need 0 < w <= k"):
        vlqadc.search_ivf_baseline(ivf, g["queries"], 0, 10)
    with pytest.raises(RuntimeError, match="search_ivf_baseline: need 0 < w <= k"):
        vlqadc.search_ivf_baseline(ivf, g["queries"], idx.k + 1, 10)
    with pytest.raises(RuntimeError, match="search_ivf_baseline: dimension mismatch"):
        vlqadc.search_ivf_baseline(ivf, np.zeros((2, idx.dim + 1), np.float32), 4, 10)
