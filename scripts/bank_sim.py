import numpy as np
z = np.load(__import__('sys').argv[1] if len(__import__('sys').argv) > 1 else 'gpurun_out/codes_c4.npz')
counts, codes = z['counts'].astype(np.int64), z['codes']
off = np.concatenate([[0], np.cumsum(counts)])
M = codes.shape[1]

def wavefronts(block):  # block: [<=32, M] codes -> mean over p of max distinct-per-bank
    tot = 0
    for p in range(M):
        c = np.unique(block[:, p])
        tot += np.bincount(c % 32, minlength=32).max()
    return tot / M

def evaluate(order_fn, U=6):
    wf, n = 0.0, 0
    for i in range(len(counts)):
        cc = codes[off[i]:off[i+1]]
        if len(cc) == 0: continue
        cc = cc[order_fn(cc)]
        # the scan: chunk of 32*U entries, lane l takes entries u*32 + l
        for s in range(0, len(cc), 32):
            blk = cc[s:s+32]
            wf += wavefronts(blk) * len(blk); n += len(blk)
    return wf / n

ident = lambda cc: np.arange(len(cc))
lex = lambda cc: np.lexsort(cc.T[::-1])
print("id order      ", round(evaluate(ident), 3))
print("lex by codes  ", round(evaluate(lex), 3))
# random model
rnd = np.random.default_rng(0).integers(0, 256, size=(32*1000, M)).astype(np.uint8)
wf = np.mean([wavefronts(rnd[s:s+32]) for s in range(0, len(rnd), 32)])
print("uniform random", round(wf, 3))
# per-subspace distinct code fraction within warps

def distinct(order_fn):
    d, n = np.zeros(M), 0
    for i in range(len(counts)):
        cc = codes[off[i]:off[i+1]]
        if len(cc) < 32: continue
        cc = cc[order_fn(cc)]
        for s in range(0, len(cc) - 31, 32):
            blk = cc[s:s+32]
            d += [len(np.unique(blk[:, p])) for p in range(M)]; n += 1
    return np.round(d / n, 1)
print("distinct/subspace id ", distinct(ident))
print("distinct/subspace lex", distinct(lex))
# greedy: order by projection onto the first principal direction of the one-hot code matrix ~ sort by tuple of (code_p) for the
# 4 lowest-entropy subspaces first
def ent_order(cc):
    ent = [len(np.unique(cc[:, p])) for p in range(M)]
    pri = np.argsort(ent)
    return np.lexsort(cc[:, pri].T[::-1])
print("entropy-lex          ", round(evaluate(ent_order), 3), distinct(ent_order))
