"""The reference's own Python smoke suite (proj/tests/python/test_smoke.py),
replayed against the drop-in module: train/add/search/save/load on the GPU."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def vlqadc():
    import torch
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    from paper_1901_00275_b200 import vlqadc as mod
    return mod


@pytest.fixture(scope="module")
def data(vlqadc):
    base = vlqadc.gen_synthetic(5000, 16, clusters=20, spread=0.05, seed=42)
    queries = vlqadc.gen_synthetic(50, 16, clusters=20, spread=0.05, seed=43)
    return base, queries


@pytest.fixture(scope="module")
def index(vlqadc, data):
    base, _ = data
    idx = vlqadc.Index.train(base, k=32, n=8, m=4, iters=8, seed=1)
    idx.add(base)
    return idx


def test_index_properties(data, index):
    base, _ = data
    assert (index.k, index.n, index.m, index.dim, index.ntotal) == (32, 8, 4, 16, len(base))


def test_search_returns_near_neighbors(vlqadc, data, index):
    base, queries = data
    gt = vlqadc.brute_force_gt(base, queries, 10)
    ids, dists = index.search(queries, w1=16, alpha=0.5, k=10)
    assert ids.shape == (50, 10) and dists.shape == (50, 10)
    assert ids.dtype == np.int64 and dists.dtype == np.float32
    assert np.all(np.diff(dists, axis=1) >= 0)
    recall = np.mean([gt[q, 0] in ids[q] for q in range(len(queries))])
    assert recall > 0.8


def test_exhaustive_search_finds_stored_points(data, index):
    base, _ = data
    ids10, _ = index.search(base[:20], w1=32, alpha=1.0, k=10)
    assert sum(q in ids10[q] for q in range(20)) >= 18


def test_save_load_roundtrip(vlqadc, tmp_path, data, index):
    _, queries = data
    path = str(tmp_path / "smoke.vlq")
    index.save(path)
    loaded = vlqadc.Index.load(path)
    a_ids, a_d = index.search(queries, w1=8, alpha=0.5, k=5)
    b_ids, b_d = loaded.search(queries, w1=8, alpha=0.5, k=5)
    assert np.array_equal(a_ids, b_ids) and np.array_equal(a_d, b_d)


def test_gpu_trained_model_is_searched_like_the_reference(vlqadc, tmp_path, data, index, oracle_mod):
    """A GPU-trained index exported as VLQ1 searches identically in the oracle."""
    _, queries = data
    path = str(tmp_path / "gpu_trained.vlq")
    index.save(path)
    o = oracle_mod.OracleIndex.load(path)
    for w1, alpha, k in [(8, 0.5, 5), (32, 1.0, 10), (4, 0.25, 100)]:
        ids, dists = index.search(queries, w1=w1, alpha=alpha, k=k)
        oids, od, _ = o.search(queries, w1, alpha, k)
        assert np.array_equal(ids, oids) and np.array_equal(dists.view(np.uint32), od.view(np.uint32))


def test_train_unclamped_and_graph_invariants(vlqadc, data, oracle_mod, tmp_path):
    base, queries = data
    idx = vlqadc.Index.train(base, k=24, n=5, m=8, iters=4, seed=7, clamp_lambda=False)
    idx.add(base)
    lo, hi = idx.lambda_range
    assert lo < hi
    path = str(tmp_path / "u.vlq")
    idx.save(path)
    from oracle import vlq1
    ix = vlq1.read(path)
    # graph rows ascending by (dist, id), no self loops, exact edge lengths
    for i in range(ix.k):
        d = ix.elen[i]
        assert np.all(d > 0) and i not in ix.nbr[i]
        assert all((d[j], ix.nbr[i, j]) <= (d[j + 1], ix.nbr[i, j + 1]) for j in range(ix.n - 1))
        all_d = ((ix.centroids[i] - ix.centroids) ** 2).sum(1)
        all_d[i] = np.inf
        assert set(np.argsort(all_d, kind="stable")[: ix.n]) == set(ix.nbr[i])
    # the add that produced this file equals the oracle's build on the same model
    model = vlq1.Vlq1(ix.dim, ix.k, ix.n, ix.m, ix.clamp, 0.0, 1.0, ix.centroids, ix.nbr, ix.elen, ix.pq)
    built = oracle_mod.OracleIndex(model).build(base)
    assert (np.float32(built.lo), np.float32(built.hi)) == (np.float32(lo), np.float32(hi))
    assert np.array_equal(built.ids, ix.ids) and np.array_equal(built.codes, ix.codes)
    assert np.array_equal(built.lambdas, ix.lambdas)


def test_errors_surface_as_exceptions(vlqadc, tmp_path):
    with pytest.raises(RuntimeError):
        vlqadc.read_vecs(str(tmp_path / "missing.fvecs"))
    with pytest.raises(RuntimeError, match="m must divide the vector dimension"):
        vlqadc.Index.train(np.zeros((10, 16), np.float32), k=4, m=3)
    with pytest.raises(RuntimeError, match="need at least k training points"):
        vlqadc.Index.train(np.zeros((10, 16), np.float32), k=40, m=4)


def test_set_max_threads_keeps_results_identical(vlqadc, data, index):
    _, queries = data
    vlqadc.set_max_threads(1)
    a_ids, _ = index.search(queries, w1=8, alpha=0.5, k=5)
    vlqadc.set_max_threads(0)
    b_ids, _ = index.search(queries, w1=8, alpha=0.5, k=5)
    assert np.array_equal(a_ids, b_ids)


def test_device_synthetic_generator_law(vlqadc):
    import torch
    n, d = 20000, 16
    x = torch.empty((n, d), dtype=torch.float32, device="cuda")
    vlqadc.gen_synthetic_device(0, n, d, 10, 0.05, 42, x.data_ptr())
    y = torch.empty((100, d), dtype=torch.float32, device="cuda")
    vlqadc.gen_synthetic_device(500, 100, d, 10, 0.05, 42, y.data_ptr())
    torch.cuda.synchronize()
    assert torch.equal(x[500:600], y)  # counter-based: rows regenerate independently
    xs = x.cpu().numpy()
    assert 0.0 < xs.mean() < 1.0 and np.isfinite(xs).all()


def test_streamed_synthetic_add_equals_host_add(vlqadc, data):
    import torch
    base, _ = data
    n, d = 30000, 16
    x = torch.empty((n, d), dtype=torch.float32, device="cuda")
    vlqadc.gen_synthetic_device(0, n, d, 20, 0.05, 5, x.data_ptr())
    torch.cuda.synchronize()
    a = vlqadc.Index.train(base, k=32, n=8, m=4, iters=3, seed=2)
    b = vlqadc.Index.train(base, k=32, n=8, m=4, iters=3, seed=2)
    a.add(x.cpu().numpy())
    b.add_synthetic(n, clusters=20, spread=0.05, seed=5)
    la, lb = a.lists(), b.lists()
    for u, v in zip(la, lb):
        assert np.array_equal(u, v)


def test_concurrent_search_on_one_index(vlqadc, data, index):
    """Index.search is const in the reference and runs with the GIL released
    (bindings.cpp:99-126, :107): several host threads may search one index at
    once.  The engine serialises the calls (per-engine mutex in the C ABI);
    every thread's result must equal the sequential one bit for bit."""
    import threading

    base, queries = data
    rng = np.random.default_rng(7)
    batches = [np.ascontiguousarray(base[rng.integers(0, len(base), 300 + 37 * t)]) for t in range(4)]
    params = [(16, 0.5, 10), (8, 0.25, 5), (32, 1.0, 20), (4, 0.5, 1)]
    expect = [index.search(b, w1=w1, alpha=a, k=k) for b, (w1, a, k) in zip(batches, params)]
    got = [[] for _ in range(4)]
    errors = []

    def worker(t):
        try:
            w1, a, k = params[t]
            for _ in range(12):
                got[t].append(index.search(batches[t], w1=w1, alpha=a, k=k))
        except Exception as e:  # surfaced below
            errors.append(e)

    threads = [threading.Thread(target=worker, args=(t,)) for t in range(4)]
    for th in threads:
        th.start()
    for th in threads:
        th.join()
    assert not errors, errors
    for t in range(4):
        assert len(got[t]) == 12
        for ids, d in got[t]:
            assert np.array_equal(ids, expect[t][0])
            assert np.array_equal(d.view(np.uint32), expect[t][1].view(np.uint32))


def test_failed_add_leaves_lambda_range_unchanged(vlqadc, data):
    """A failing add must not alter the index (the reference assigns the
    index only after build_index succeeds, bindings.cpp:89-96)."""
    base, _ = data
    idx = vlqadc.Index.train(base, k=32, n=8, m=4, iters=4, seed=3, clamp_lambda=False)
    before = idx.lambda_range
    with pytest.raises(RuntimeError, match="dimension mismatch"):
        idx.add(np.zeros((0, 5), np.float32))
    assert idx.lambda_range == before and idx.ntotal == 0
    # a degenerate edge (c == 0) fails the encode pass AFTER the unclamped
    # model's observe_lambda_range pre-pass has run
    mdl = idx.model()
    elen = mdl["elen"].copy()
    elen[:, :] = 0.0
    bad = vlqadc.Index.from_model(mdl["dim"], mdl["k"], mdl["n"], mdl["m"], False, 0.25, 0.75, mdl["centroids"],
                                  mdl["nbr"], elen, mdl["pq"])
    with pytest.raises(RuntimeError, match="degenerate edge"):
        bad.add(base)
    assert bad.lambda_range == (0.25, 0.75) and bad.ntotal == 0
    idx.add(base)
    assert idx.ntotal == len(base)


def test_get_cells_equals_slices_of_the_full_lists(index):
    """vlq_engine_get_cells (sampled add replay at 1e9 entries) returns exactly
    the requested slices of vlq_engine_get_lists, in request order."""
    off, ids, codes, lams = index.lists()
    rng = np.random.default_rng(3)
    req = rng.integers(0, index.k * index.n, size=40).astype(np.uint32)
    req[5] = req[6]  # duplicates are allowed
    counts, cids, ccodes, clams = index.cells(req)
    pos = 0
    for i, c in enumerate(req):
        a, b = int(off[c]), int(off[c + 1])
        assert counts[i] == b - a
        assert np.array_equal(cids[pos:pos + b - a], ids[a:b])
        assert np.array_equal(ccodes[pos:pos + b - a], codes[a:b])
        assert np.array_equal(clams[pos:pos + b - a], lams[a:b])
        pos += b - a
    assert pos == len(cids)
    with pytest.raises(RuntimeError, match="out of range"):
        index.cells([index.k * index.n])
