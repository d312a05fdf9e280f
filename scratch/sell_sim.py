# Lane efficiency of length-sorted lane-per-row SpMV layouts on the C4 graph (R-MAT s22 ef16),
# counted on the CPU from the oracle's CSR.  A "window" of W consecutive rows is sorted by row
# length (groups of 4 entries); rows longer than T groups go to warp-cooperative processing; the
# rest are cut into 32-row slices whose cost is 32 x (longest row of the slice) lane-groups.
# Efficiency = groups actually stored / lane-groups issued.
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import oracle

scale = int(sys.argv[1]) if len(sys.argv) > 1 else 22
src, dst = oracle.rmat_edges(scale, 16, 1)
n = 1 << scale
rp, ci, deg = oracle.build_csr(n, src, dst)
L = np.diff(rp)
g = (L + 3) // 4
print(f"n {n} nnz {ci.shape[0]} groups {g.sum()} empty rows {(L == 0).sum()} max row {L.max()}")
for q in (1, 2, 4, 8, 16, 32, 64, 128, 512, 2048):
    sel = g > q
    print(f"  rows > {q:5d} groups: {sel.sum():8d}  their groups {g[sel].sum() / g.sum() * 100:5.1f} %")


def sim(W, T):
    nw = (n + W - 1) // W
    gp = np.zeros(nw * W, np.int64)
    gp[:n] = g
    gw = gp.reshape(nw, W)
    long_ = gw > T
    gs = np.where(long_, 0, gw)
    gs = -np.sort(-gs, axis=1)                       # descending inside the window
    sl = gs.reshape(nw, W // 32, 32)
    cost = sl[:, :, 0].sum() * 32                     # lane-groups of the short slices
    eff = gs.sum() / max(cost, 1)
    lg = gw[long_]
    lcost = ((lg + 31) // 32 * 32).sum()              # warp-per-row: 32 groups per step
    leff = lg.sum() / max(lcost, 1)
    tot = (gs.sum() + lg.sum()) / (cost + lcost)
    print(f"W {W:8d} T {T:4d}: short eff {eff:.3f} ({gs.sum()/1e6:.2f} M groups)  long rows {long_.sum():7d} eff {leff:.3f}"
          f"  overall {tot:.3f}  warp-steps {(cost + lcost) / 32 / 1e6:.2f} M")


for W in (128, 1024, 4096, 1 << 16, n):
    for T in (8, 16, 32, 64):
        sim(W, T)
