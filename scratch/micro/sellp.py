import numpy as np
def build(rp, ci, deg, LONG=2048, LCAP=16, CH=2048, NWT=148 * 32, MLP=16, RMAX=8):
    """SELL-P-pow2 plan (numpy reference of the GPU plan builder)."""
    n = len(rp) - 1
    order = np.argsort(-deg.astype(np.int64), kind='stable'); cperm = np.empty(n, np.int64); cperm[order] = np.arange(n)
    ncols = int((deg > 0).sum())
    g = (cperm[ci] + 1).astype(np.int64)            # gather index, 0 = zero column
    lens = np.diff(rp).astype(np.int64)
    rowP = np.argsort(-lens, kind='stable')          # P-order: longest first
    lP = lens[rowP]
    nlong = int((lP > LONG).sum()); nempty0 = int(np.searchsorted(-lP, 0, side='left'))   # first empty P index
    # groups
    mid = np.arange(nlong, nempty0)
    lm = lP[mid]
    gl = np.zeros(len(mid), np.int64)
    for e in range(6):
        gg = 1 << e
        sel = (gl == 0) & (((lm + gg - 1) // gg <= LCAP) | (gg == 32))
        gl[sel] = gg
    # slices: consecutive rows with same g; g == 1 slices hold R rows per lane (R * L <= MLP)
    per = (lm + gl - 1) // gl
    sl_base, sl_g, sl_nr, sl_R, sl_L = [], [], [], [], []
    q = 0
    while q < len(mid):
        gg = gl[q]
        if gg == 1:
            L0 = per[q]; R = max(1, min(RMAX, MLP // max(L0, 1)))
            rps = 32 * R
        else:
            R = 1; rps = 32 // gg
        e = q
        while e < len(mid) and e - q < rps and gl[e] == gg: e += 1
        sl_base.append(nlong + q); sl_g.append(gg); sl_nr.append(e - q); sl_R.append(R); sl_L.append(per[q:e].max()); q = e
    sl_base = np.array(sl_base, np.int64); sl_g = np.array(sl_g, np.int64); sl_nr = np.array(sl_nr, np.int64)
    sl_R = np.array(sl_R, np.int64); Ls = np.array(sl_L, np.int64)
    ns = len(sl_base)
    sid_of_row = np.repeat(np.arange(ns), sl_nr)
    soff = np.r_[0, np.cumsum(32 * Ls * sl_R)][:-1]
    idx = np.zeros(int((32 * Ls * sl_R).sum()), np.int32)
    rows_nat = rowP[mid]
    E = lm
    rep = np.repeat(np.arange(len(mid)), E)
    j = np.arange(int(E.sum())) - np.repeat(np.cumsum(E) - E, E)
    gg = gl[rep]; s = sid_of_row[rep]
    slot = (nlong + np.arange(len(mid)))[rep] - sl_base[s]           # row slot in slice
    # g == 1: slot = r * 32 + lane ; entry k of row r of lane at [r][k][lane]
    RR = sl_R[s]; LL = Ls[s]
    lane = np.where(gg == 1, slot % 32, slot * gg + (j % gg))
    r = np.where(gg == 1, slot // 32, 0)
    k = np.where(gg == 1, j, j // gg)
    idx[soff[s] + 32 * (r * LL + k) + lane] = g[rp[rows_nat[rep]] + j]
    # chunks for long rows (P-order first)
    chunks = []; longs = []; tot = 0
    for qq in range(nlong):
        row = rowP[qq]; p0, p1 = rp[row], rp[row + 1]; nch = (p1 - p0 + CH - 1) // CH
        longs.append((qq, tot, nch, 0))
        for u in range(nch):
            pb = p0 + u * CH; chunks.append((qq, pb & 0xffffffff, pb >> 32, min(CH, p1 - pb)))
        tot += nch
    chunks = np.array(chunks, np.int64).astype(np.uint32).view(np.int32).reshape(-1, 4) if chunks else np.zeros((0, 4), np.int32)
    longs = np.array(longs, np.int32).reshape(-1, 4)
    # warp ranges over slices, balanced by entries
    w = 32 * Ls * sl_R + 16 * sl_R + 32
    cw = np.r_[0, np.cumsum(w)]
    wt = np.searchsorted(cw, np.linspace(0, cw[-1], NWT + 1), side='left').astype(np.int32); wt[-1] = ns
    hdr = np.stack([soff, sl_base, Ls | (sl_R << 16), np.log2(sl_g).astype(np.int64) | (sl_nr << 8)], 1).astype(np.int64)
    gposP = np.where(deg[rowP] > 0, cperm[rowP] + 1, -1).astype(np.int32)
    return dict(n=n, ncols=ncols, nslices=ns, nlong=nlong, nempty0=nempty0, idx=idx, hdr=hdr, wt=wt, chunks=chunks, longs=longs,
                rowP=rowP, gposP=gposP, cperm=cperm, Ls=Ls)

def emulate(p, yg1, rp, ci):
    """row sums in P order (mid rows only)"""
    out = np.zeros(p['n'])
    for s in range(p['nslices']):
        off, base, LR, gn = p['hdr'][s]; L = LR & 0xffff; R = LR >> 16; lg = gn & 0xff; nr = gn >> 8; gg = 1 << lg
        blk = p['idx'][off: off + 32 * L * R].reshape(R, L, 32)
        vals = yg1[blk].astype(np.float64).sum(1)     # [R][32]
        if gg == 1:
            for q in range(nr): out[base + q] = vals[q // 32, q % 32]
        else:
            for q in range(nr): out[base + q] = vals[0, q * gg:(q + 1) * gg].sum()
    return out
