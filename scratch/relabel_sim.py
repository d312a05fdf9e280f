# VERDICT r1 item 4(i)/(iii) on the C4 graph, counted on the CPU (oracle CSR): what a
# locality-preserving relabel (columns bucketed by floor(log2 count), original id order inside a
# bucket) does to the sweep's cold gathers, and how many hot-cache bank conflicts replicating the
# hottest columns would remove.  Per warp step of 256 consecutive entries (the skeleton's 64-group
# step): cold entries, distinct cold 32-byte sectors (what L2 serves), distinct 128-byte lines
# (what the L1TEX t-stage processes per instruction, roughly); hot lookups and bank conflicts.
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import oracle

scale = int(sys.argv[1]) if len(sys.argv) > 1 else 22
src, dst = oracle.rmat_edges(scale, 16, 1)
n = 1 << scale
rp, ci, deg = oracle.build_csr(n, src, dst)
nnz = ci.shape[0]
cnt = np.bincount(ci, minlength=n)
nz = np.nonzero(cnt)[0]
HC = 168 * 1024 // 4                      # hot-cache entries (fp32)
step = np.arange(nnz, dtype=np.int64) // 256


def layout(key):
    order = nz[np.lexsort((nz, key))]      # key ascending, ties by id
    pos = np.empty(n, np.int64)
    pos[order] = np.arange(order.shape[0])
    return pos[ci]


def stats(name, p, hc=HC, R=0):
    hot = p < hc
    cold = ~hot
    sc, pc = step[cold], p[cold]
    sectors = np.unique(sc * (1 << 26) + pc // 8).shape[0]
    lines = np.unique(sc * (1 << 26) + pc // 32).shape[0]
    # bank conflicts of hot lookups per 32-lane instruction (32 consecutive hot entries): extra
    # wavefronts = max over banks of the distinct words it is asked for - 1.  A replicated column
    # (position < R, one copy per bank) is read by lane l from bank l.
    ph = p[hot]
    m = (ph.shape[0] // 32) * 32
    w = ph[:m].reshape(-1, 32).copy()
    lane = np.broadcast_to(np.arange(32), w.shape)
    rep = w < R
    bank = np.where(rep, lane, w % 32)
    word = np.where(rep, (1 << 40) + w * 32 + lane, w)
    worst = np.zeros(w.shape[0], np.int64)
    for b in range(32):
        sel = np.where(bank == b, word, -1)
        sel.sort(axis=1)
        distinct = ((np.diff(sel, axis=1) != 0) & (sel[:, 1:] >= 0)).sum(axis=1) + (sel[:, 0] >= 0)
        distinct = np.where((sel[:, 0] < 0) & (sel[:, -1] >= 0), distinct + 1, distinct)
        worst = np.maximum(worst, distinct)
    extra = int((worst - 1).clip(min=0).sum())
    print(f"{name:38s} hot {hot.mean()*100:5.1f}%  cold entries {cold.sum()/1e6:6.2f} M  cold sectors {sectors/1e6:6.2f} M  "
          f"cold lines {lines/1e6:6.2f} M  hot-LDS extra wavefronts {extra/1e6:5.2f} M")


print(f"R-MAT s{scale} ef16: n {n}, nnz {nnz}, non-empty columns {nz.shape[0]}, hot cache {HC} entries")
stats("degree-sorted (product)", layout(-cnt[nz]))
stats("log2-bucketed, id order inside", layout(-np.floor(np.log2(cnt[nz])).astype(np.int64)))
# bank replication of the R hottest columns (one copy per bank): the replicas cost 31 R entries of
# hot capacity
p0 = layout(-cnt[nz])
for R in (64, 256, 1024):
    stats(f"degree-sorted, top {R} replicated x32", p0, hc=HC - 31 * R, R=R)
