import sys, numpy as np, torch
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tests")
from conftest import load_golden
from paper_1901_00275_b200 import vlqadc
from paper_1901_00275_b200 import dist as vdist
from oracle import oracle
z, index_path, _ = load_golden("accept_small")
q = torch.from_numpy(z["queries"]).cuda(); nq = q.shape[0]
st = torch.cuda.current_stream().cuda_stream
o = oracle.OracleIndex.load(index_path)
full = vlqadc.Index.load(index_path)
G = 3
shards = [vlqadc.Index.load(index_path, shard_rank=r, shard_count=G) for r in range(G)]
for w1, alpha, k in [(16, 0.5, 10), (64, 0.25, 100)]:
    oids, od, _ = o.search(z["queries"], w1, alpha, k)
    fi, fd = full.search(z["queries"], w1=w1, alpha=alpha, k=k)
    print("full==oracle", np.array_equal(fi, oids))
    otop = np.sort(o.first_level(z["queries"], w1), 1)
    tops = []
    for r in range(G):
        lo, hi = vdist.query_slice(nq, r, G)
        t = torch.empty((hi - lo, w1), dtype=torch.int32, device="cuda")
        shards[r].search_coarse_device(q[lo:hi].data_ptr(), hi - lo, w1, t.data_ptr(), st)
        tops.append(t)
    top = torch.cat(tops).contiguous()
    gt = np.sort(top.cpu().numpy().view(np.uint32), 1)
    print(w1, "sliced coarse sets == oracle", np.array_equal(gt, otop), np.where((gt != otop).any(1))[0][:10])
    pi, pd = [], []
    for s in shards:
        ids = torch.empty((nq, k), dtype=torch.int64, device="cuda")
        d = torch.empty((nq, k), dtype=torch.float32, device="cuda")
        s.search_fine_device(q.data_ptr(), nq, w1, alpha, k, top.data_ptr(), ids.data_ptr(), d.data_ptr(), None, st)
        pi.append(ids); pd.append(d)
    for r, s in enumerate(shards):
        ids2, d2 = s.search(z["queries"], w1=w1, alpha=alpha, k=k)
        a = pi[r].cpu().numpy()
        print(" shard", r, "fine==own full search", np.array_equal(a, ids2), np.where((a != ids2).any(1))[0][:10])
    gi, gd = vdist.merge_topk(torch.stack(pi), torch.stack(pd))
    print(w1, "merged==oracle", np.array_equal(gi.cpu().numpy(), oids))
