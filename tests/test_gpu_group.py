"""The multi-GPU group (vlq_group_*, csrc/group.cu) on one B200: G shard
engines listed on the same device exercise the whole schedule -- query-split
selection, the sharded scan reading each query's selection from the engine
that made it (peer-pointer loads; local here), and the per-slice merge of
every shard's top-k -- and must return the single engine's / the
reference's results bit for bit."""
import numpy as np
import pytest

from conftest import ALL_CASES, grid_of, load_golden, regen_base

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def vlqadc():
    import torch
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    from paper_1901_00275_b200 import vlqadc as mod
    return mod


def same_f32(a, b):
    return np.array_equal(np.asarray(a, np.float32).view(np.uint32), np.asarray(b, np.float32).view(np.uint32))


@pytest.mark.parametrize("G,S", [(1, 0), (2, 0), (3, 0), (5, 0), (4, 2), (6, 3), (4, 1), (8, 2)])
@pytest.mark.parametrize("name", ["accept_small", "m16", "unclamped"])
def test_group_search_matches_reference_golden(vlqadc, name, G, S):
    """G members as G / S replicas of an S-way list sharding (S = 0: G)."""
    z, index_path, _ = load_golden(name)
    grp = vlqadc.IndexGroup.load(index_path, [0] * G, shards=S)
    assert len(grp) == G and grp.replicas * grp.shards == G
    ent = grp.local_entries()
    for r in range(grp.replicas):  # every replica holds the whole index, split into its shards
        assert sum(ent[r * grp.shards:(r + 1) * grp.shards]) == grp.ntotal
    for gi, (w1, alpha, k) in enumerate(grid_of(z)):
        ids, dists, scanned = grp.search(z["queries"], w1=w1, alpha=alpha, k=k, return_scanned=True)
        assert np.array_equal(ids, z[f"ids_{gi}"]), (name, G, gi)
        assert same_f32(dists, z[f"dists_{gi}"]), (name, G, gi)
        assert int(scanned.sum()) == int(z[f"scanned_{gi}"]), (name, G, gi)


def test_group_add_and_resident_search_match_single_engine(vlqadc, oracle_mod):
    z, index_path, model_path = load_golden("m16")
    base = regen_base(z)
    single = vlqadc.Index.load(model_path)
    single.add(base)
    model = single.model()
    grp = vlqadc.IndexGroup.from_model(model, [0, 0, 0, 0, 0, 0], shards=3)
    grp.add(base)
    assert grp.ntotal == single.ntotal
    o = oracle_mod.OracleIndex.load(index_path)
    rng = np.random.default_rng(5)
    for _ in range(4):
        w1 = int(rng.integers(1, single.k + 1))
        alpha = float(np.float32(rng.uniform(0.05, 1.0)))
        k = int(rng.choice([1, 10, 100]))
        a_ids, a_d, a_sc = single.search(z["queries"], w1=w1, alpha=alpha, k=k, return_scanned=True)
        b_ids, b_d, b_sc = grp.search(z["queries"], w1=w1, alpha=alpha, k=k, return_scanned=True)
        assert np.array_equal(a_ids, b_ids) and same_f32(a_d, b_d) and np.array_equal(a_sc, b_sc)
        oids, od, _ = o.search(z["queries"], w1, alpha, k)
        assert np.array_equal(b_ids, oids) and same_f32(b_d, od)
    # device-resident batch + timed searches
    grp.set_queries(z["queries"])
    ms = grp.search_resident(16, 0.5, 10)
    assert ms > 0
    r_ids, r_d, r_sc = grp.results()
    a_ids, a_d, a_sc = single.search(z["queries"], w1=16, alpha=0.5, k=10, return_scanned=True)
    assert np.array_equal(r_ids, a_ids) and same_f32(r_d, a_d) and np.array_equal(r_sc, a_sc)


def test_group_tensor_core_chunk_select_path(vlqadc, oracle_mod, tmp_path, monkeypatch):
    """K = 16384, n = 32, D = 96: every member's selection runs the
    chunk-select tensor-core coarse stage with the select-split hand-off."""
    base = vlqadc.gen_synthetic(30000, 96, clusters=3000, spread=0.05, seed=55)
    q = vlqadc.gen_synthetic(77, 96, clusters=3000, spread=0.05, seed=56)
    idx = vlqadc.Index.train(base, k=16384, n=32, m=16, iters=2, seed=8)
    idx.add(base)
    path = str(tmp_path / "g16k.vlq")
    idx.save(path)
    o = oracle_mod.OracleIndex.load(path)
    grp = vlqadc.IndexGroup.load(path, [0, 0, 0, 0], shards=2)
    for w1, alpha, k in [(64, 0.25, 100), (16, 0.5, 10), (200, 0.1, 20)]:
        ids, d = grp.search(q, w1=w1, alpha=alpha, k=k)
        oids, od, _ = o.search(q, w1, alpha, k)
        assert np.array_equal(ids, oids) and same_f32(d, od), (w1, alpha, k)


def test_group_errors(vlqadc):
    z, index_path, _ = load_golden("accept_small")
    grp = vlqadc.IndexGroup.load(index_path, [0, 0])
    with pytest.raises(RuntimeError, match="first_level_scan: need 0 < w1 <= k"):
        grp.search(z["queries"], w1=grp.info().k + 1, alpha=0.5, k=10)
    with pytest.raises(RuntimeError, match="dimension mismatch"):
        grp.search(np.zeros((3, grp.info().dim + 1), np.float32), w1=4, alpha=0.5, k=10)
    with pytest.raises(RuntimeError, match="device index out of range"):
        vlqadc.IndexGroup([0, 99])
    with pytest.raises(RuntimeError, match="shards must divide"):
        vlqadc.IndexGroup([0, 0, 0], shards=2)
    with pytest.raises(RuntimeError, match="index already holds a base set"):
        grp.add(regen_base(z))


@pytest.mark.parametrize("k", [1500])
def test_group_large_k_and_exact_scan(vlqadc, oracle_mod, k):
    """k > 1024 (every shard's exact all-candidates path, merged by the group)
    and the forced exact scan through a 3-shard group."""
    z, index_path, _ = load_golden("m16")
    o = oracle_mod.OracleIndex.load(index_path)
    for kw in [dict(), dict(force_exact=True)]:
        grp = vlqadc.IndexGroup.load(index_path, [0, 0, 0], **kw)
        for w1, alpha, kk in [(16, 0.5, k), (8, 1.0, 100)]:
            ids, d = grp.search(z["queries"][:30], w1=w1, alpha=alpha, k=kk)
            oids, od, _ = o.search(z["queries"][:30], w1, alpha, kk)
            assert np.array_equal(ids, oids) and same_f32(d, od), (kw, w1, alpha, kk)
