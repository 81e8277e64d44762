"""Tensor-core (tcgen05 TF32) coarse stage and add assignment, forced on for
the small golden models (VLQ_TC_MIN_K=0): results must stay bit-exact with
the reference -- the TF32 candidates are only proposals, settled by exact
reference-order distances under a certificate."""
import numpy as np
import pytest

from conftest import grid_of, load_golden, regen_base

pytestmark = pytest.mark.gpu

# golden cases whose dim is a multiple of 8 (the tf32 MMA K step)
TC_CASES = ["smoke", "unclamped", "m16", "n1m8", "accept_small"]


@pytest.fixture()
def vlqadc(monkeypatch):
    import torch
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    monkeypatch.setenv("VLQ_TC_MIN_K", "0")
    monkeypatch.setenv("VLQ_TC", "1")
    from paper_1901_00275_b200 import vlqadc as mod
    return mod


def same_f32(a, b):
    return np.array_equal(np.asarray(a, np.float32).view(np.uint32), np.asarray(b, np.float32).view(np.uint32))


@pytest.mark.parametrize("name", TC_CASES)
def test_tc_search_matches_reference_golden(vlqadc, name):
    z, index_path, _ = load_golden(name)
    idx = vlqadc.Index.load(index_path)
    for gi, (w1, alpha, k) in enumerate(grid_of(z)):
        ids, dists, scanned = idx.search(z["queries"], w1=w1, alpha=alpha, k=k, return_scanned=True)
        assert np.array_equal(ids, z[f"ids_{gi}"]), (name, gi)
        assert same_f32(dists, z[f"dists_{gi}"]), (name, gi)
        assert int(scanned.sum()) == int(z[f"scanned_{gi}"]), (name, gi)


@pytest.mark.parametrize("name", [c for c in TC_CASES if c != "accept_small"])
def test_tc_add_matches_reference_file(vlqadc, name, tmp_path):
    z, index_path, model_path = load_golden(name)
    base = regen_base(z)
    idx = vlqadc.Index.load(model_path)
    idx.add(base)
    out = str(tmp_path / "tc.vlq")
    idx.save(out)
    assert open(out, "rb").read() == open(index_path, "rb").read()


def test_tc_per_point_assignment_matches_oracle(vlqadc, oracle_mod):
    z, index_path, _ = load_golden("accept_small")
    base = regen_base(z)
    idx = vlqadc.Index.load(index_path)
    cells, lams, codes, lb = idx.encode(base)
    oc, ol, ocd, olb = oracle_mod.OracleIndex.load(index_path).assign(base)
    assert np.array_equal(cells, oc) and same_f32(lams, ol)
    assert np.array_equal(codes, ocd) and np.array_equal(lb, olb)


def test_tc_random_parameters_match_oracle(vlqadc, oracle_mod):
    rng = np.random.default_rng(7)
    for name in TC_CASES:
        z, index_path, _ = load_golden(name)
        idx = vlqadc.Index.load(index_path)
        o = oracle_mod.OracleIndex.load(index_path)
        for _ in range(4):
            w1 = int(rng.integers(1, idx.k))
            alpha = float(np.float32(rng.uniform(0.05, 1.0)))
            k = int(rng.choice([1, 10, 100]))
            ids, dists = idx.search(z["queries"], w1=w1, alpha=alpha, k=k)
            oids, od, _ = o.search(z["queries"], w1, alpha, k)
            assert np.array_equal(ids, oids) and same_f32(dists, od), (name, w1, alpha, k)


def test_tc_larger_codebook_trained_on_gpu(vlqadc, oracle_mod, tmp_path):
    """K = 2048 GPU-trained model (D = 32): tensor-core add + search vs the
    oracle on the exported file."""
    base = vlqadc.gen_synthetic(60000, 32, clusters=300, spread=0.05, seed=5)
    q = vlqadc.gen_synthetic(200, 32, clusters=300, spread=0.05, seed=6)
    idx = vlqadc.Index.train(base[:20000], k=2048, n=16, m=8, iters=4, seed=3)
    idx.add(base)
    path = str(tmp_path / "k2048.vlq")
    idx.save(path)
    o = oracle_mod.OracleIndex.load(path)
    built = o.build(base)  # the oracle's own add on the same model
    off, ids, codes, lams = idx.lists()
    assert np.array_equal(off, built.list_off) and np.array_equal(ids, built.ids)
    assert np.array_equal(codes, built.codes) and np.array_equal(lams, built.lambdas)
    for w1, alpha, k in [(64, 0.25, 100), (16, 0.5, 10), (256, 0.1, 50)]:
        ids_, d_ = idx.search(q, w1=w1, alpha=alpha, k=k)
        oids, od, _ = o.search(q, w1, alpha, k)
        assert np.array_equal(ids_, oids) and same_f32(d_, od)


@pytest.mark.parametrize("store_rows", ["0", "1"])
def test_tc_two_pass_coarse_filter_large_k(vlqadc, oracle_mod, tmp_path, monkeypatch, store_rows):
    """K = 16384: the two-pass tensor-core coarse stage (chunk minima -> tau ->
    filtered candidate list, no K-wide rows in HBM) and the store-rows variant
    both reproduce the oracle exactly."""
    monkeypatch.setenv("VLQ_TC_STORE_ROWS", store_rows)
    base = vlqadc.gen_synthetic(120000, 32, clusters=2000, spread=0.05, seed=15)
    q = vlqadc.gen_synthetic(150, 32, clusters=2000, spread=0.05, seed=16)
    idx = vlqadc.Index.train(base[:60000], k=16384, n=8, m=8, iters=3, seed=4)
    idx.add(base)
    path = str(tmp_path / "k16k.vlq")
    idx.save(path)
    o = oracle_mod.OracleIndex.load(path)
    for w1, alpha, k in [(16, 0.5, 10), (64, 0.25, 100), (200, 0.1, 20)]:
        ids_, d_ = idx.search(q, w1=w1, alpha=alpha, k=k)
        oids, od, _ = o.search(q, w1, alpha, k)
        assert np.array_equal(ids_, oids) and same_f32(d_, od), (w1, alpha, k)


@pytest.mark.parametrize("dim", [96, 128])
def test_tc_two_pass_coarse_filter_deep_dims(vlqadc, oracle_mod, tmp_path, dim):
    """The C4 (D = 96, 3xTF32: hi + lo tiles) and C3/C5 (D = 128) shapes of
    the two-pass coarse stage: the shared-memory ring depth is chosen to fit
    227 KB, and the result stays bit-exact with the oracle."""
    base = vlqadc.gen_synthetic(40000, dim, clusters=1500, spread=0.05, seed=25)
    q = vlqadc.gen_synthetic(120, dim, clusters=1500, spread=0.05, seed=26)
    idx = vlqadc.Index.train(base[:30000], k=4096, n=8, m=8, iters=2, seed=4)
    idx.add(base)
    path = str(tmp_path / f"d{dim}.vlq")
    idx.save(path)
    o = oracle_mod.OracleIndex.load(path)
    # persistent / per-row-block coarse grids, 1xTF32 first pass, scan variants
    variants = [dict(tc_persist=1), dict(tc_persist=0), dict(tc_pass1_single=1),
                dict(tc_pass1_single=1, tc_persist=0), dict(tc_chunk_select=0), dict(tc_chunk_select=0, tc_persist=0),
                dict(tc_chunk_cap=4), dict(tc_center=0),
                dict(scan_packed=0), dict(scan_slots=104), dict(scan_slots=4), dict(scan_slots=8),
                dict(scan_slots=6), dict(scan_slots=306),
                dict(tc_chunk_select=0, tc_pass1_single=1, tc_pass2_single=1),
                dict(tc_chunk_select=0, tc_pass1_single=1, tc_pass2_single=1, tc_persist=0),
                dict(cert_slack_milli=10**6, scan_retry=0), dict(cert_slack_milli=10**6)]
    for v in variants:
        knobs = dict(tc_persist=1, tc_pass1_single=0, tc_chunk_select=1, tc_chunk_cap=256, tc_center=1,
                     scan_slots=0, scan_packed=1,
                     tc_pass2_single=0, scan_retry=1, cert_slack_milli=0)
        knobs.update(v)
        for key, val in knobs.items():
            idx.set_tuning(key, val)
        for w1, alpha, k in [(16, 0.5, 10), (64, 0.25, 100)]:
            ids_, d_ = idx.search(q, w1=w1, alpha=alpha, k=k)
            oids, od, _ = o.search(q, w1, alpha, k)
            assert np.array_equal(ids_, oids) and same_f32(d_, od), (dim, v, w1, alpha, k)


@pytest.mark.parametrize("dim,m", [(96, 16), (128, 8)])
def test_tc_add_lists_and_search_at_baseline_shapes(vlqadc, oracle_mod, tmp_path, dim, m):
    """BASELINE shapes (C4: D = 96, m = 16; C3/C5: D = 128, m = 8) with
    n = 32 edges and K = 16384, tensor cores forced: the GPU add (TF32
    ARGMIN proposals + certificate-checked exact refine) builds the same
    lists as the oracle's build_index, point for point, and the 3xTF32 coarse
    search returns the oracle's ids and distances."""
    base = vlqadc.gen_synthetic(40000, dim, clusters=4000, spread=0.05, seed=35)
    q = vlqadc.gen_synthetic(64, dim, clusters=4000, spread=0.05, seed=36)
    idx = vlqadc.Index.train(base, k=16384, n=32, m=m, iters=2, seed=6)
    idx.add(base)
    path = str(tmp_path / f"bl{dim}.vlq")
    idx.save(path)
    o = oracle_mod.OracleIndex.load(path)
    built = o.build(base)
    off, ids, codes, lams = idx.lists()
    assert np.array_equal(off, built.list_off) and np.array_equal(ids, built.ids)
    assert np.array_equal(codes, built.codes) and np.array_equal(lams, built.lambdas)
    # the add path's per-point outputs on held-out points (the certificate at D = 96 / 128)
    extra = vlqadc.gen_synthetic(3000, dim, clusters=4000, spread=0.05, seed=37)
    cells, lam, cd, lb = idx.encode(extra)
    oc, ol, ocd, olb = o.assign(extra)
    assert np.array_equal(cells, oc) and same_f32(lam, ol)
    assert np.array_equal(cd, ocd) and np.array_equal(lb, olb)
    for w1, alpha, k in [(64, 0.25, 100), (16, 1.0, 10)]:
        ids_, d_ = idx.search(q, w1=w1, alpha=alpha, k=k)
        oids, od, _ = o.search(q, w1, alpha, k)
        assert np.array_equal(ids_, oids) and same_f32(d_, od), (dim, w1, alpha, k)


@pytest.mark.parametrize("dim", [96, 128])
def test_chunk_select_coarse_stage_paths_match_oracle(vlqadc, oracle_mod, tmp_path, dim):
    """The chunk-select coarse stage (select_fused.cu: one 1xTF32 pass of
    8-centroid chunk minima, exact evaluation of the chunks within the TF32
    bound, fused first + second level) at K = 16384, n = 32: bit-exact with the
    oracle through its normal path, through the exact full-row fallback
    (chunk list capped below w1, so every query overflows), and equal to the
    two-pass filter path it replaces; the select-split hand-off (cells + exact
    (a, b)) of the fused kernel feeds a second engine's fine stage."""
    base = vlqadc.gen_synthetic(40000, dim, clusters=3000, spread=0.05, seed=45)
    q = vlqadc.gen_synthetic(96, dim, clusters=3000, spread=0.05, seed=46)
    idx = vlqadc.Index.train(base, k=16384, n=32, m=8, iters=2, seed=7)
    idx.add(base)
    path = str(tmp_path / f"cs{dim}.vlq")
    idx.save(path)
    o = oracle_mod.OracleIndex.load(path)
    grid = [(64, 0.25, 100), (16, 0.5, 10), (200, 0.1, 20), (1, 1.0, 5)]
    ref = {g: o.search(q, g[0], g[1], g[2])[:2] for g in grid}
    idx.set_profiling(True)
    for knobs in [dict(tc_chunk_select=1, tc_chunk_cap=256), dict(tc_chunk_select=1, tc_chunk_cap=4),
                  dict(tc_chunk_select=1, tc_chunk_cap=256, tc_center=0), dict(tc_persist=0),
                  dict(tc_persist=1, tc_center=1, tc_chunk_select=0)]:
        for key, val in knobs.items():
            idx.set_tuning(key, val)
        for g in grid:
            ids_, d_ = idx.search(q, w1=g[0], alpha=g[1], k=g[2])
            oids, od = ref[g]
            assert np.array_equal(ids_, oids) and same_f32(d_, od), (dim, knobs, g)
        st = idx.stats(reset=True)
        if knobs.get("tc_chunk_cap") == 4:
            assert st["tc_fallbacks"] > 0  # the fallback path really ran
    idx.set_tuning("tc_chunk_select", 1)
    idx.set_tuning("tc_chunk_cap", 256)
    # select-split: this engine selects, a second engine on the same model scans
    import torch
    dq = torch.from_numpy(q).cuda()
    w1, alpha, k = 64, 0.25, 100
    w2 = idx.w2(w1, alpha)
    sel = torch.empty((len(q), w2), dtype=torch.int32, device="cuda")
    ab = torch.empty((len(q), w2, 2), dtype=torch.float32, device="cuda")
    idx.search_select_device(dq.data_ptr(), len(q), w1, alpha, sel.data_ptr(), ab.data_ptr(), stream=0)
    other = vlqadc.Index.load(path)
    other.set_tuning("tc_chunk_select", 0)
    ids = torch.empty((len(q), k), dtype=torch.int64, device="cuda")
    dd = torch.empty((len(q), k), dtype=torch.float32, device="cuda")
    sc = torch.empty((len(q),), dtype=torch.int64, device="cuda")
    other.search_fine_sel_device(dq.data_ptr(), len(q), w1, alpha, k, sel.data_ptr(), ab.data_ptr(), ids.data_ptr(),
                                 dd.data_ptr(), sc.data_ptr(), stream=0)
    torch.cuda.synchronize()
    oids, od = ref[(w1, alpha, k)]
    assert np.array_equal(ids.cpu().numpy(), oids) and same_f32(dd.cpu().numpy(), od)


@pytest.mark.parametrize("dim", [96, 128])
def test_chunk_select_centered_operands_on_offset_data(vlqadc, oracle_mod, tmp_path, dim):
    """Data far from the origin (every coordinate + 40): the TF32 bound of the
    uncentered chunk pass grows with |y| |c| until every query overflows its
    chunk list and takes the exact full-row fallback; on centered operands
    (queries and centroids minus the centroid mean) the bound is that of the
    data's spread, no query falls back, and both stay bit-exact with the
    oracle."""
    base = vlqadc.gen_synthetic(40000, dim, clusters=3000, spread=0.05, seed=55) + np.float32(40.0)
    q = vlqadc.gen_synthetic(96, dim, clusters=3000, spread=0.05, seed=56) + np.float32(40.0)
    idx = vlqadc.Index.train(base, k=16384, n=32, m=8, iters=2, seed=8)
    idx.add(base)
    path = str(tmp_path / f"off{dim}.vlq")
    idx.save(path)
    o = oracle_mod.OracleIndex.load(path)
    idx.set_profiling(True)
    fallbacks = {}
    for center in (1, 0):
        idx.set_tuning("tc_center", center)
        idx.stats(reset=True)
        for w1, alpha, k in [(64, 0.25, 100), (16, 0.5, 10)]:
            ids_, d_ = idx.search(q, w1=w1, alpha=alpha, k=k)
            oids, od, _ = o.search(q, w1, alpha, k)
            assert np.array_equal(ids_, oids) and same_f32(d_, od), (dim, center, w1)
        fallbacks[center] = idx.stats(reset=True)["tc_fallbacks"]
    assert fallbacks[1] == 0 and fallbacks[0] > 0, fallbacks
