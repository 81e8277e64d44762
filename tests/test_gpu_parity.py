"""GPU parity tests: the CUDA engine (libvlqgpu.so through the C ABI) against
the reference's golden outputs and the C oracle, bit-exact.

Parity bar (BASELINE.json north_star): ids and PQ codes bit-exact; distances
within 1e-4 relative.  The engine reproduces the reference's fp32 operation
order, so every check below is exact equality (a stricter bar)."""
import os
import subprocess

import numpy as np
import pytest

from conftest import ALL_CASES, PY_CASES, ROOT, grid_of, load_golden, regen_base

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def vlqadc():
    import torch
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    from paper_1901_00275_b200 import vlqadc as mod
    return mod


def same_f32(a, b):
    return np.array_equal(np.asarray(a, np.float32).view(np.uint32), np.asarray(b, np.float32).view(np.uint32))


@pytest.mark.parametrize("name", ALL_CASES)
@pytest.mark.parametrize("force_exact", [False, True])
def test_search_matches_reference_golden(vlqadc, name, force_exact):
    z, index_path, _ = load_golden(name)
    idx = vlqadc.Index.load(index_path, force_exact=force_exact)
    for gi, (w1, alpha, k) in enumerate(grid_of(z)):
        ids, dists, scanned = idx.search(z["queries"], w1=w1, alpha=alpha, k=k, return_scanned=True)
        assert np.array_equal(ids, z[f"ids_{gi}"]), (name, gi)
        assert same_f32(dists, z[f"dists_{gi}"]), (name, gi)
        assert int(scanned.sum()) == int(z[f"scanned_{gi}"]), (name, gi)


@pytest.mark.parametrize("name", PY_CASES)
def test_add_matches_reference_lists_and_file(vlqadc, name, tmp_path):
    """Index.load(model) + add(base) == the reference-built index, byte for
    byte after save (lists, lambda bytes, codes, t3, header)."""
    z, index_path, model_path = load_golden(name)
    base = regen_base(z)
    idx = vlqadc.Index.load(model_path)
    assert idx.ntotal == 0
    idx.add(base)
    assert idx.ntotal == len(base)
    out = str(tmp_path / "gpu.vlq")
    idx.save(out)
    assert open(out, "rb").read() == open(index_path, "rb").read()
    # and it searches exactly like the reference
    for gi, (w1, alpha, k) in enumerate(grid_of(z)):
        ids, dists = idx.search(z["queries"], w1=w1, alpha=alpha, k=k)
        assert np.array_equal(ids, z[f"ids_{gi}"]) and same_f32(dists, z[f"dists_{gi}"])


def test_add_per_point_replay_matches_oracle(vlqadc, oracle_mod):
    """Per-point (cell, exact lambda, code, lambda byte): test_index.cpp:161-189."""
    z, index_path, model_path = load_golden("accept_small")
    base = regen_base(z)
    idx = vlqadc.Index.load(index_path)
    cells, lams, codes, lb = idx.encode(base)
    o = oracle_mod.OracleIndex.load(index_path)
    oc, ol, ocd, olb = o.assign(base)
    assert np.array_equal(cells, oc)
    assert same_f32(lams, ol)
    assert np.array_equal(codes, ocd)
    assert np.array_equal(lb, olb)


def test_exhaustive_search_equals_full_scan(vlqadc, oracle_mod):
    """w1 = K, alpha = 1 (test_search.cpp:286-313, acceptance C3)."""
    z, index_path, _ = load_golden("accept_small")
    idx = vlqadc.Index.load(index_path)
    o = oracle_mod.OracleIndex.load(index_path)
    q = z["queries"][:20]
    for k in (1, 10, 100):
        ids, dists = idx.search(q, w1=idx.k, alpha=1.0, k=k)
        oids, odists, _ = o.search(q, idx.k, 1.0, k)
        assert np.array_equal(ids, oids) and same_f32(dists, odists)


@pytest.mark.parametrize("seed,knobs", [(0, {}), (1, {}), (2, {"scan_slots": 8}), (3, {"scan_variant": 1}),
                                        (4, {"scan_slots": 104}), (5, {"cert_slack_milli": 10**6}),
                                        (6, {"scan_relabel": 0}), (7, {"scan_reorder": 0})])
def test_random_parameters_match_oracle(vlqadc, oracle_mod, seed, knobs):
    """Random (w1, alpha, k) vs the oracle: the fused fast scan (6 / 8 / 4
    slots per lane, 3 or 4 CTAs per SM), the generic warp-buffer scan, and a widened
    certificate that sends every query through the retry pass and the exact
    scan, the scan copy without its code relabeling and the canonical arrays
    -- results must not change."""
    rng = np.random.default_rng(seed)
    for name in ALL_CASES:
        z, index_path, _ = load_golden(name)
        idx = vlqadc.Index.load(index_path)
        for key, val in knobs.items():
            idx.set_tuning(key, val)
        o = oracle_mod.OracleIndex.load(index_path)
        for _ in range(3):
            w1 = int(rng.integers(1, idx.k + 1))
            alpha = float(np.float32(rng.uniform(0.01, 1.0)))
            k = int(rng.choice([1, 3, 10, 64, 100, 300]))
            ids, dists, sc = idx.search(z["queries"], w1=w1, alpha=alpha, k=k, return_scanned=True)
            oids, od, osc = o.search(z["queries"], w1, alpha, k)
            assert np.array_equal(ids, oids), (name, w1, alpha, k)
            assert same_f32(dists, od)
            assert np.array_equal(sc, osc)


def test_padding_and_short_results(vlqadc, oracle_mod):
    """S_q < k -> padded with -1 / +inf (bindings.cpp:116-124)."""
    z, index_path, _ = load_golden("m1")
    idx = vlqadc.Index.load(index_path)
    ids, dists = idx.search(z["queries"], w1=1, alpha=0.01, k=1000)
    oids, od, _ = oracle_mod.OracleIndex.load(index_path).search(z["queries"], 1, 0.01, 1000)
    assert np.array_equal(ids, oids) and same_f32(dists, od)
    assert (ids == -1).any() and np.isinf(dists[ids == -1]).all()


def test_errors_mirror_reference(vlqadc, tmp_path):
    z, index_path, model_path = load_golden("smoke")
    idx = vlqadc.Index.load(index_path)
    q = z["queries"]
    with pytest.raises(RuntimeError, match="first_level_scan: need 0 < w1 <= k"):
        idx.search(q, w1=0)
    with pytest.raises(RuntimeError, match="first_level_scan: need 0 < w1 <= k"):
        idx.search(q, w1=idx.k + 1)
    with pytest.raises(RuntimeError, match="dimension mismatch"):
        idx.search(np.zeros((3, idx.dim + 1), np.float32))
    with pytest.raises(RuntimeError, match="expected a 2-D float array"):
        idx.search(np.zeros(16, np.float32))
    with pytest.raises(RuntimeError, match="non-finite"):
        idx.search(np.full((2, 16), np.nan, np.float32))
    with pytest.raises(RuntimeError, match="index already holds a base set"):
        idx.add(q)
    bad = tmp_path / "bad.vlq"
    raw = open(index_path, "rb").read()
    bad.write_bytes(b"XXXX" + raw[4:])
    with pytest.raises(RuntimeError, match="bad magic"):
        vlqadc.Index.load(str(bad))
    bad.write_bytes(raw[: len(raw) // 2])
    with pytest.raises(RuntimeError, match="truncated"):
        vlqadc.Index.load(str(bad))
    with pytest.raises(RuntimeError, match="cannot open"):
        vlqadc.Index.load(str(tmp_path / "missing.vlq"))
    m = vlqadc.Index.load(model_path)
    with pytest.raises(RuntimeError, match="build_index: empty base set"):
        m.add(np.zeros((0, 16), np.float32))


def test_degenerate_edge_raises(vlqadc):
    """line_lambda throws on c <= 0 (line_quant.cpp:10-12)."""
    from oracle import vlq1
    _, _, model_path = load_golden("smoke")
    mdl = vlq1.read(model_path)
    elen = mdl.elen.copy()
    elen[0, 0] = 0.0
    idx = vlqadc.Index.from_model(mdl.dim, mdl.k, mdl.n, mdl.m, mdl.clamp, mdl.lo, mdl.hi, mdl.centroids, mdl.nbr,
                                  elen, mdl.pq)
    with pytest.raises(RuntimeError, match="degenerate edge"):
        idx.search(mdl.centroids[:4], w1=mdl.k, alpha=1.0, k=5)


def test_single_point_base(vlqadc, oracle_mod):
    """test_search.cpp:316-330: a one-point base returns that point."""
    z, _, model_path = load_golden("m1")
    idx = vlqadc.Index.load(model_path)
    idx.add(np.array([[0.5, 0.25, -0.5, 1.0]], np.float32))
    ids, dists = idx.search(np.full((1, 4), 0.1, np.float32), w1=idx.k, alpha=1.0, k=5)
    assert ids[0, 0] == 0 and (ids[0, 1:] == -1).all()


def test_centroids_land_in_own_region_rank0(vlqadc):
    """test_index.cpp:138-159."""
    from oracle import vlq1
    _, _, model_path = load_golden("smoke")
    mdl = vlq1.read(model_path)
    idx = vlqadc.Index.load(model_path)
    cells, lams, _, lb = idx.encode(mdl.centroids)
    assert np.array_equal(cells, np.arange(mdl.k) * mdl.n)
    assert (lb == 0).all()


def test_identical_queries_identical_results(vlqadc):
    z, index_path, _ = load_golden("smoke")
    idx = vlqadc.Index.load(index_path)
    q = np.repeat(z["queries"][5:6], 3, axis=0)
    ids, dists = idx.search(q, w1=8, alpha=0.5, k=10)
    assert (ids == ids[0]).all() and (dists == dists[0]).all()


def test_tiling_independence(vlqadc):
    """Results do not depend on the query tile size (determinism contract,
    README.md:55-56)."""
    z, index_path, _ = load_golden("accept_small")
    a = vlqadc.Index.load(index_path)
    b = vlqadc.Index.load(index_path, max_tile=7)
    for w1, alpha, k in [(16, 0.5, 10), (64, 0.25, 100)]:
        ia, da = a.search(z["queries"], w1=w1, alpha=alpha, k=k)
        ib, db = b.search(z["queries"], w1=w1, alpha=alpha, k=k)
        assert np.array_equal(ia, ib) and same_f32(da, db)


def test_brute_force_gt_matches_reference(vlqadc):
    z, _, _ = load_golden("smoke")
    base = regen_base(z)
    gt = vlqadc.brute_force_gt(base, z["queries"], 10)
    assert np.array_equal(gt, z["gt10"])


def test_sharded_engines_merge_to_the_single_engine_result(vlqadc):
    """Lists sharded by region over 3 engines on one device; the (dist, id)
    merge (K9) of per-shard top-k equals the unsharded result."""
    import torch
    from paper_1901_00275_b200 import dist as vdist
    z, index_path, _ = load_golden("accept_small")
    full = vlqadc.Index.load(index_path)
    shards = [vlqadc.Index.load(index_path, shard_rank=r, shard_count=3) for r in range(3)]
    assert sum(s.local_entries for s in shards) == full.ntotal
    for w1, alpha, k in [(16, 0.5, 10), (64, 0.25, 100)]:
        want_ids, want_d = full.search(z["queries"], w1=w1, alpha=alpha, k=k)
        parts = [s.search(z["queries"], w1=w1, alpha=alpha, k=k) for s in shards]
        pi = torch.from_numpy(np.stack([p[0] for p in parts])).cuda()
        pd = torch.from_numpy(np.stack([p[1] for p in parts])).cuda()
        got_i, got_d = vdist.merge_topk(pi, pd)
        assert np.array_equal(got_i.cpu().numpy(), want_ids)
        assert same_f32(got_d.cpu().numpy(), want_d)


@pytest.mark.parametrize("tc", ["0", "1"])
def test_query_split_staged_search_matches_single_engine(vlqadc, monkeypatch, tc):
    """The multi-GPU schedule on one device: the coarse stage
    (search_coarse_device) runs per query slice, the slices' top-w1 tables
    are concatenated, every shard engine runs search_fine_device on the whole
    batch, and the K9 merge equals the unsharded search bit-exactly (with the
    tensor-core coarse stage forced on and off)."""
    import torch
    from paper_1901_00275_b200 import dist as vdist
    monkeypatch.setenv("VLQ_TC_MIN_K", "0" if tc == "1" else "100000000")
    z, index_path, _ = load_golden("accept_small")
    full = vlqadc.Index.load(index_path)
    G = 3
    shards = [vlqadc.Index.load(index_path, shard_rank=r, shard_count=G) for r in range(G)]
    q = torch.from_numpy(z["queries"]).cuda()
    nq = q.shape[0]
    st = torch.cuda.current_stream().cuda_stream
    for w1, alpha, k in [(16, 0.5, 10), (64, 0.25, 100), (5, 1.0, 7)]:
        want_ids, want_d = full.search(z["queries"], w1=w1, alpha=alpha, k=k)
        tops = []
        for r in range(G):
            lo, hi = vdist.query_slice(nq, r, G)
            t = torch.empty((hi - lo, w1), dtype=torch.int32, device="cuda")
            if hi > lo:
                shards[r].search_coarse_device(q[lo:hi].data_ptr(), hi - lo, w1, t.data_ptr(), st)
            tops.append(t)
        top = torch.cat(tops).contiguous()
        pi, pd = [], []
        for s in shards:
            ids = torch.empty((nq, k), dtype=torch.int64, device="cuda")
            d = torch.empty((nq, k), dtype=torch.float32, device="cuda")
            s.search_fine_device(q.data_ptr(), nq, w1, alpha, k, top.data_ptr(), ids.data_ptr(), d.data_ptr(),
                                 None, st)
            pi.append(ids)
            pd.append(d)
        got_i, got_d = vdist.merge_topk(torch.stack(pi), torch.stack(pd))
        for s in shards:
            s.sync(st)
        assert np.array_equal(got_i.cpu().numpy(), want_ids), (w1, alpha, k)
        assert same_f32(got_d.cpu().numpy(), want_d), (w1, alpha, k)


@pytest.mark.parametrize("tc", ["0", "1"])
def test_select_split_staged_search_matches_single_engine(vlqadc, oracle_mod, monkeypatch, tc):
    """The select-split multi-GPU schedule on one device: first level + cell
    selection (search_select_device) per query slice, the slices' cells and
    (a, b) pairs concatenated, every shard engine runs search_fine_sel_device
    on the whole batch, and the K9 merge equals the unsharded search
    bit-exactly; the hand-off equals the oracle's (select())."""
    import torch
    from paper_1901_00275_b200 import dist as vdist
    monkeypatch.setenv("VLQ_TC_MIN_K", "0" if tc == "1" else "100000000")
    z, index_path, _ = load_golden("accept_small")
    full = vlqadc.Index.load(index_path)
    o = oracle_mod.OracleIndex.load(index_path)
    G = 3
    shards = [vlqadc.Index.load(index_path, shard_rank=r, shard_count=G) for r in range(G)]
    q = torch.from_numpy(z["queries"]).cuda()
    nq = q.shape[0]
    st = torch.cuda.current_stream().cuda_stream
    for w1, alpha, k in [(16, 0.5, 10), (64, 0.25, 100), (5, 1.0, 7)]:
        want_ids, want_d = full.search(z["queries"], w1=w1, alpha=alpha, k=k)
        w2 = full.w2(w1, alpha)
        sels, abs_ = [], []
        for r in range(G):
            lo, hi = vdist.query_slice(nq, r, G)
            sl = torch.empty((hi - lo, w2), dtype=torch.int32, device="cuda")
            ab = torch.empty((hi - lo, w2, 2), dtype=torch.float32, device="cuda")
            if hi > lo:
                shards[r].search_select_device(q[lo:hi].data_ptr(), hi - lo, w1, alpha, sl.data_ptr(), ab.data_ptr(),
                                               st)
            sels.append(sl)
            abs_.append(ab)
        sel = torch.cat(sels).contiguous()
        ab = torch.cat(abs_).contiguous()
        osel, oab = o.select(z["queries"], w1, alpha)
        torch.cuda.synchronize()
        # the same cell SET per query (the engine lists it by edge position,
        # the oracle by distance), with the same (a, b) for each cell
        gsel, gab = sel.cpu().numpy().view(np.uint32), ab.cpu().numpy()
        gi_, oi_ = np.argsort(gsel, axis=1), np.argsort(osel, axis=1)
        assert np.array_equal(np.take_along_axis(gsel, gi_, 1), np.take_along_axis(osel, oi_, 1))
        assert same_f32(np.take_along_axis(gab, gi_[:, :, None], 1), np.take_along_axis(oab, oi_[:, :, None], 1))
        pi, pd = [], []
        for s in shards:
            ids = torch.empty((nq, k), dtype=torch.int64, device="cuda")
            d = torch.empty((nq, k), dtype=torch.float32, device="cuda")
            s.search_fine_sel_device(q.data_ptr(), nq, w1, alpha, k, sel.data_ptr(), ab.data_ptr(), ids.data_ptr(),
                                     d.data_ptr(), None, st)
            pi.append(ids)
            pd.append(d)
        got_i, got_d = vdist.merge_topk(torch.stack(pi), torch.stack(pd))
        for s in shards:
            s.sync(st)
        assert np.array_equal(got_i.cpu().numpy(), want_ids), (w1, alpha, k)
        assert same_f32(got_d.cpu().numpy(), want_d), (w1, alpha, k)


@pytest.mark.slow
def test_acceptance_c7_trend_kats(vlqadc, tmp_path):
    """acceptance.cpp:330-363 on the reference's 'big' instance, built by the
    reference (oracle/_ref/ref_tools): recall@10 for w1 = 8/16/32/64 and the
    scanned totals for alpha = 0.25/0.40/0.50 must equal the reference's
    golden numbers."""
    tools = os.path.join(ROOT, "oracle", "_ref", "ref_tools")
    if not os.path.exists(tools):
        pytest.skip("oracle/_ref not built")
    from oracle import vlq1
    prefix = str(tmp_path / "big")
    subprocess.run([tools, "instance", "1000000", "32", "200", "1024", "16", "8", "6", "100000", "500", "2000",
                    "0.25", prefix], check=True, timeout=1500)
    idx = vlqadc.Index.load(prefix + ".vlq")
    base = vlq1.read_fvecs(prefix + ".base.fvecs")
    q = vlq1.read_fvecs(prefix + ".queries.fvecs")
    gt = vlqadc.brute_force_gt(base, q, 10)
    want_r10 = {8: 0.6700, 16: 0.7560, 32: 0.8260, 64: 0.8740}
    for w1, r10 in want_r10.items():
        ids, _ = idx.search(q, w1=w1, alpha=1.0, k=10)
        rec = np.mean([gt[i, 0] in ids[i] for i in range(len(q))])
        assert round(rec, 4) == r10, (w1, rec)
    want_scan = {0.25: 7746348, 0.4: 12339928, 0.5: 15436084}
    for alpha, total in want_scan.items():
        _, _, sc = idx.search(q, w1=64, alpha=alpha, k=10, return_scanned=True)
        assert int(sc.sum()) == total, (alpha, int(sc.sum()))


@pytest.mark.parametrize("G,k", [(2, 10), (8, 100), (3, 1), (5, 37)])
def test_merge_of_sorted_parts_random(vlqadc, G, k):
    """K9 on random sorted parts (ragged: each part holds a random number of
    real rows, -1/+inf padded; equal distances across parts broken by id)
    equals a host (dist, id) merge."""
    import torch
    from paper_1901_00275_b200 import dist as vdist
    rng = np.random.default_rng(G * 100 + k)
    nq = 64
    ids = np.full((G, nq, k), -1, np.int64)
    d = np.full((G, nq, k), np.inf, np.float32)
    perm = rng.permutation(G * nq * k)  # unique ids across parts
    for g in range(G):
        for q in range(nq):
            n = int(rng.integers(0, k + 1))
            dd = np.round(rng.uniform(0, 4, n), 1).astype(np.float32)  # many ties
            ii = perm[(g * nq + q) * k:(g * nq + q) * k + n].astype(np.int64)
            o = np.lexsort((ii, dd))
            ids[g, q, :n], d[g, q, :n] = ii[o], dd[o]
    got_i, got_d = vdist.merge_topk(torch.from_numpy(ids).cuda(), torch.from_numpy(d).cuda())
    got_i, got_d = got_i.cpu().numpy(), got_d.cpu().numpy()
    for q in range(nq):
        m = ids[:, q, :] >= 0
        ci, cd = ids[:, q, :][m], d[:, q, :][m]
        o = np.lexsort((ci, cd))[:k]
        want_i = np.full(k, -1, np.int64)
        want_d = np.full(k, np.inf, np.float32)
        want_i[:len(o)], want_d[:len(o)] = ci[o], cd[o]
        assert np.array_equal(got_i[q], want_i), q
        assert same_f32(got_d[q], want_d)


@pytest.mark.parametrize("name,suffix,chunk", [("smoke", ".fvecs", 0), ("unclamped", ".fvecs", 777),
                                                ("m16", ".bvecs", 1000), ("n1m8", ".ivecs", 0)])
def test_add_vecs_streamed_file_equals_reference_build(vlqadc, name, suffix, chunk, tmp_path):
    """Index.add_vecs(path) (streamed from the file, any chunking; unclamped
    models take two passes over the file) == add(read_vecs(path)); for the
    float file the result is the reference-built index byte for byte."""
    z, index_path, model_path = load_golden(name)
    base = regen_base(z)
    if suffix != ".fvecs":  # byte / int payloads: integer-valued data of the same shape
        base = np.clip(np.rint(base * 255.0), 0, 255).astype(np.float32)
    path = str(tmp_path / f"base{suffix}")
    vlqadc.write_vecs(base, path)
    want = vlqadc.Index.load(model_path)
    want.add(vlqadc.read_vecs(path))
    got = vlqadc.Index.load(model_path)
    got.add_vecs(path, chunk_rows=chunk)
    assert got.ntotal == len(base)
    a, b = str(tmp_path / "want.vlq"), str(tmp_path / "got.vlq")
    want.save(a)
    got.save(b)
    assert open(a, "rb").read() == open(b, "rb").read()
    if suffix == ".fvecs":
        assert open(b, "rb").read() == open(index_path, "rb").read()


def test_add_vecs_errors_mirror_read_vecs(vlqadc, tmp_path):
    z, _, model_path = load_golden("smoke")
    base = regen_base(z)[:100]
    path = str(tmp_path / "b.fvecs")
    vlqadc.write_vecs(base, path)
    raw = open(path, "rb").read()
    cases = {"missing.fvecs": None, "empty.fvecs": b"", "trunc.fvecs": raw[:-3], "hdr.fvecs": raw + b"\x01\x00"}
    msgs = {"missing.fvecs": "cannot open", "empty.fvecs": "no records", "trunc.fvecs": "truncated record payload",
            "hdr.fvecs": "truncated record header"}
    for fname, data in cases.items():
        p = str(tmp_path / fname)
        if data is not None:
            open(p, "wb").write(data)
        idx = vlqadc.Index.load(model_path)
        with pytest.raises(RuntimeError, match=msgs[fname]):
            idx.add_vecs(p)
        assert idx.ntotal == 0
    other = str(tmp_path / "d.fvecs")
    vlqadc.write_vecs(np.zeros((4, base.shape[1] + 1), np.float32), other)
    with pytest.raises(RuntimeError, match="dimension mismatch"):
        vlqadc.Index.load(model_path).add_vecs(other)
    idx = vlqadc.Index.load(model_path)
    idx.add_vecs(path)
    with pytest.raises(RuntimeError, match="index already holds a base set"):
        idx.add_vecs(path)


@pytest.mark.parametrize("retry", [0, 1])
def test_certificate_retry_and_exact_fallback_match_oracle(vlqadc, oracle_mod, retry):
    """A widened certificate (test knob cert_slack) fails for every query,
    so the retry pass (fast scan again with 4 k' for the listed queries,
    re-score) and the exact scan for what still fails both run; with the
    retry on or off the results equal the oracle's."""
    for name in ALL_CASES:
        z, index_path, _ = load_golden(name)
        idx = vlqadc.Index.load(index_path)
        idx.set_tuning("cert_slack_milli", 10**6)
        idx.set_tuning("scan_retry", retry)
        o = oracle_mod.OracleIndex.load(index_path)
        for w1, alpha, k in [(min(idx.k, 16), 0.5, 10), (min(idx.k, 64), 0.25, 100), (min(idx.k, 8), 1.0, 3)]:
            ids, dists, sc = idx.search(z["queries"], w1=w1, alpha=alpha, k=k, return_scanned=True)
            oids, od, osc = o.search(z["queries"], w1, alpha, k)
            assert np.array_equal(ids, oids), (name, w1, alpha, k)
            assert same_f32(dists, od)
            assert np.array_equal(sc, osc)


@pytest.mark.parametrize("k", [1500, 3000])
def test_large_k_matches_oracle(vlqadc, oracle_mod, k):
    """select_topk has no cap on k (search.cpp:122-140): k > 1024 takes the
    exact all-candidates path (large_k.cu: exact keys of every scanned entry,
    segmented sort per query), padded with -1 / +inf when fewer were scanned."""
    for name in ["accept_small", "m16", "smoke"]:
        z, index_path, _ = load_golden(name)
        idx = vlqadc.Index.load(index_path)
        o = oracle_mod.OracleIndex.load(index_path)
        for w1, alpha in [(min(idx.k, 16), 0.5), (idx.k, 1.0)]:
            ids, dists, sc = idx.search(z["queries"][:40], w1=w1, alpha=alpha, k=k, return_scanned=True)
            oids, od, osc = o.search(z["queries"][:40], w1, alpha, k)
            assert np.array_equal(ids, oids), (name, w1, alpha, k)
            assert same_f32(dists, od)
            assert np.array_equal(sc, osc)
