# Offline model of the fast scan's LUT bank conflicts under a per-sub-space code
# relabeling (co-occurrence partition, as engine.cu choose_code_banks): train on a
# fraction of the dumped lists (scripts/code_dump.py), evaluate on the rest.
# usage: python scripts/bank_perm_sim.py 0.85
import numpy as np, sys
z = np.load('gpurun_out/codes_c4.npz')
counts, codes = z['counts'].astype(np.int64), z['codes']
off = np.concatenate([[0], np.cumsum(counts)])
M = codes.shape[1]
L = len(counts)
lists = [codes[off[i]:off[i+1]] for i in range(L)]
rng = np.random.default_rng(1)
idx = rng.permutation(L); cut = int(L*float(sys.argv[1])); tr, te = idx[:cut], idx[cut:]
lex = lambda cc: np.lexsort(cc.T[::-1])
def blocks(sel):
    for i in sel:
        cc = lists[i]
        if len(cc)==0: continue
        cc = cc[lex(cc)]
        for s in range(0, len(cc), 32):
            yield cc[s:s+32]
def evaluate(sel, perm):  # perm[p][c] -> slot (0..255); bank = slot % 32
    wf=n=0
    for blk in blocks(sel):
        t=0
        for p in range(M):
            c = np.unique(blk[:,p]); t += np.bincount(perm[p][c] % 32, minlength=32).max()
        wf += t/M*len(blk); n += len(blk)
    return wf/n
ident = np.tile(np.arange(256), (M,1))
print('identity train/test', evaluate(tr, ident), evaluate(te, ident))
# frequency round-robin
freq = np.zeros((M,256))
co = np.zeros((M,256,256))
for blk in blocks(tr):
    w = len(blk)
    for p in range(M):
        c = np.unique(blk[:,p])
        freq[p, c] += w
        co[p][np.ix_(c,c)] += w
rr = np.zeros((M,256),dtype=np.int64)
for p in range(M):
    order = np.argsort(-freq[p])
    slot = np.zeros(256, dtype=np.int64)
    for r, c in enumerate(order):
        slot[c] = (r % 32) + 32 * (r // 32)
    rr[p] = slot
print('freq-rr  train/test', evaluate(tr, rr), evaluate(te, rr))
# greedy partition on co-occurrence then local swaps
gp = np.zeros((M,256),dtype=np.int64)
for p in range(M):
    C = co[p].copy(); np.fill_diagonal(C, 0)
    bank = -np.ones(256, dtype=np.int64); size = np.zeros(32, dtype=np.int64)
    cost = np.zeros((256,32))
    for c in np.argsort(-freq[p]):
        cand = np.where(size < 8)[0]
        b = cand[np.argmin(cost[c, cand])]
        bank[c] = b; size[b] += 1
        cost[:, b] += C[:, c]
    # local search: swaps
    for it in range(3):
        improved = 0
        for a in range(256):
            for b2 in range(a+1, 256):
                ba, bb = bank[a], bank[b2]
                if ba == bb: continue
                # delta of moving a->bb and b2->ba
                d = (cost[a,bb]-C[a,b2]) - cost[a,ba] + (cost[b2,ba]-C[b2,a]) - cost[b2,bb]
                if d < -1e-9:
                    cost[:, ba] += -C[:, a] + C[:, b2]; cost[:, bb] += -C[:, b2] + C[:, a]
                    bank[a], bank[b2] = bb, ba; improved += 1
        if not improved: break
    slot = np.zeros(256, dtype=np.int64); cnt = np.zeros(32, dtype=np.int64)
    for c in range(256):
        slot[c] = bank[c] + 32*cnt[bank[c]]; cnt[bank[c]] += 1
    gp[p] = slot
print('co-part  train/test', evaluate(tr, gp), evaluate(te, gp))
