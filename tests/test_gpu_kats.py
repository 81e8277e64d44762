"""The reference's hand-made known-answer tests (proj/tests/*.cpp) run through
the CUDA path: constructed ties and exact hits on the tensor-core ARGMIN /
chunk-select coarse stage and on the fast scan's and the exact scan's
selections."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(params=["cuda_cores", "tensor_cores"])
def vlqadc(request, monkeypatch):
    import torch
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    if request.param == "tensor_cores":
        monkeypatch.setenv("VLQ_TC_MIN_K", "0")
        monkeypatch.setenv("VLQ_TC", "1")
    else:
        monkeypatch.setenv("VLQ_TC_MIN_K", "100000000")
    from paper_1901_00275_b200 import vlqadc as mod
    return mod


def model_from_centroids(vlqadc, cent, n, m=1, seed=0):
    """A VLQ1 model over given centroids: exact n-NN graph, squared edge
    lengths, a simple PQ codebook."""
    k, dim = cent.shape
    d2 = ((cent[:, None, :].astype(np.float64) - cent[None, :, :]) ** 2).sum(-1)
    np.fill_diagonal(d2, np.inf)
    nbr = np.argsort(d2, axis=1, kind="stable")[:, :n].astype(np.uint32)
    elen = np.array([[np.float32(((cent[i] - cent[j]) ** 2).sum()) for j in nbr[i]] for i in range(k)], np.float32)
    rng = np.random.default_rng(seed)
    pq = (rng.standard_normal((m, 256, dim // m)) * 0.01).astype(np.float32)
    return vlqadc.Index.from_model(dim, k, n, m, True, 0.0, 1.0, cent, nbr, elen, pq)


def test_assign_nearest_equidistant_tie_goes_to_lowest_id(vlqadc):
    """test_quantizers.cpp:85-94: centroids {10, 20, 3, 30, 40, 50, 5} on a
    line, x = 4 is at distance 1 from centroids 2 and 6 -> id 2 (embedded in
    D = 8 so the tensor-core assignment runs too)."""
    line = np.array([10, 20, 3, 30, 40, 50, 5], np.float32)
    cent = np.zeros((7, 8), np.float32)
    cent[:, 0] = line
    idx = model_from_centroids(vlqadc, cent, n=2, m=1)
    x = np.zeros((3, 8), np.float32)
    x[:, 0] = 4.0
    cells, lams, codes, lb = idx.encode(x)
    assert np.all(cells // idx.n == 2)


def test_first_level_query_at_a_centroid(vlqadc):
    """test_search.cpp:72-76: a query equal to centroid 9 has it as its
    nearest region (w1 = 1), on the exact and the tensor-core coarse stages."""
    rng = np.random.default_rng(3)
    cent = rng.random((64, 8), dtype=np.float32)
    idx = model_from_centroids(vlqadc, cent, n=4, m=2)
    import torch
    q = torch.from_numpy(np.ascontiguousarray(cent[[9, 9, 17, 63]])).cuda()
    top = torch.empty((4, 1), dtype=torch.int32, device="cuda")
    idx.search_coarse_device(q.data_ptr(), 4, 1, top.data_ptr(), 0)
    torch.cuda.synchronize()
    assert top[:, 0].cpu().tolist() == [9, 9, 17, 63]


@pytest.mark.parametrize("force_exact", [False, True])
def test_select_topk_equal_distances_order_by_ascending_id(vlqadc, force_exact):
    """test_search.cpp:262-267: candidates tied at equal distance come out by
    ascending id -- here three identical base vectors (ids 3, 7, 9) answer a
    query at that vector with k = 2: [3, 7] (fast scan + re-score, and the
    exact scan)."""
    rng = np.random.default_rng(11)
    base = (rng.random((12, 8), dtype=np.float32) * 4.0).astype(np.float32)
    base[7] = base[3]
    base[9] = base[3]
    idx = vlqadc.Index.train(np.vstack([base, rng.random((400, 8), dtype=np.float32) * 4.0]), k=16, n=4, m=2,
                             iters=4, seed=5, force_exact=force_exact)
    idx.add(base)
    ids, dists = idx.search(base[3:4], w1=16, alpha=1.0, k=2)
    assert ids[0].tolist() == [3, 7]
    assert dists[0, 0] == dists[0, 1]
    ids3, _ = idx.search(base[3:4], w1=16, alpha=1.0, k=3)
    assert ids3[0].tolist() == [3, 7, 9]
