import numpy as np
def build(rp, ci, deg, SB=15, LM=256, nctas=148):
    n = len(rp) - 1; nnz = len(ci)
    order = np.argsort(-deg.astype(np.int64), kind='stable'); perm = np.empty(n, np.int64); perm[order] = np.arange(n)
    ncols = int((deg > 0).sum())
    g = perm[ci]
    lens = np.diff(rp); row = np.repeat(np.arange(n, dtype=np.int64), lens)
    b = g >> SB
    key = b * (n + 1) + row
    idx = np.argsort(key, kind='stable')             # entries by (block, row, position)
    ks = key[idx]
    brk = np.flatnonzero(np.r_[True, ks[1:] != ks[:-1]])
    pstart = brk; pcnt = np.diff(np.r_[brk, nnz])
    pblk = ks[brk] // (n + 1); prow = ks[brk] % (n + 1)
    # sub-pairs
    nsub = (pcnt + LM - 1) // LM
    sp_pair = np.repeat(np.arange(len(pcnt)), nsub)
    sp_k = np.arange(len(sp_pair)) - np.repeat(np.cumsum(nsub) - nsub, nsub)
    sp_start = pstart[sp_pair] + sp_k * LM
    sp_len = np.minimum(LM, pcnt[sp_pair] - sp_k * LM)
    sp_blk = pblk[sp_pair]; sp_row = prow[sp_pair]
    # slots: order (row, block, k)
    so_ = np.lexsort((sp_k, sp_blk, sp_row))
    slot = np.empty(len(so_), np.int64); slot[so_] = np.arange(len(so_))
    rslot = np.zeros(n + 1, np.int64); np.add.at(rslot, sp_row + 1, 1); rslot = np.cumsum(rslot)
    # SELL order: by block, then len desc (stable)
    sel = np.lexsort((-sp_len, sp_blk))
    nb = int(b.max()) + 1 if nnz else 0
    # pad each block's sub-pair list to a multiple of 32
    blk_sorted = sp_blk[sel]
    bounds = np.searchsorted(blk_sorted, np.arange(nb + 1))
    cnt_b = np.diff(bounds); nq_b = (cnt_b + 31) // 32
    # padded SELL position of each sub-pair in sel order
    pad_before = np.r_[0, np.cumsum(nq_b * 32 - cnt_b)][:-1]
    pos = np.arange(len(sel)) + np.repeat(pad_before, cnt_b)
    tot = int((nq_b * 32).sum())
    L = np.zeros(tot, np.int64); L[pos] = sp_len[sel]
    st = np.zeros(tot, np.int64); st[pos] = sp_start[sel]
    sslot = -np.ones(tot, np.int64); sslot[pos] = slot[sel]
    nq = tot // 32
    sl = L.reshape(nq, 32).max(1)
    so = np.r_[0, np.cumsum(32 * sl)][:-1]
    sb = np.repeat(np.arange(nb), nq_b)
    # entries
    E = int(L.sum())
    lane_pos = np.repeat(np.arange(tot), L)
    kk = np.arange(E) - np.repeat(np.cumsum(L) - L, L)
    dstpos = so[lane_pos // 32] + 32 * kk + (lane_pos % 32)
    lcol = np.zeros(int(32 * sl.sum()), np.uint16)
    lcol[dstpos] = (g[idx[st[lane_pos] + kk]] & ((1 << SB) - 1)).astype(np.uint16)
    sb = sb.astype(np.int32); so = so.astype(np.int64); sl = sl.astype(np.int32)
    slen = L.astype(np.uint16)
    sslot = sslot.astype(np.int32)
    # CTA partition by padded entries
    w = 32 * sl.astype(np.int64) + 64
    cw = np.r_[0, np.cumsum(w)]
    cs = np.searchsorted(cw, np.linspace(0, cw[-1], nctas + 1), side='left').astype(np.int32)
    cs[-1] = len(sl)
    gpos = np.where(deg > 0, perm, -1).astype(np.int32)
    return dict(n=n, ncols=ncols, SB=SB, cs=cs, sb=sb, so=so, sl=sl, sslot=sslot, slen=slen, lcol=lcol,
                rslot=rslot.astype(np.int32), gpos=gpos, nslots=len(slot), perm=perm)

def emulate(p, y_g):
    part = np.zeros(p['nslots'])
    S = 1 << p['SB']
    for q in range(len(p['sl'])):
        b = p['sb'][q]; L = p['sl'][q]; off = p['so'][q]
        blk = p['lcol'][off:off + 32 * L].reshape(L, 32)
        for j in range(32):
            s = p['sslot'][32 * q + j]
            if s < 0: continue
            lj = p['slen'][32 * q + j]
            part[s] = np.sum(y_g[b * S + blk[:lj, j].astype(np.int64)].astype(np.float64))
    n = p['n']
    out = np.array([part[p['rslot'][i]:p['rslot'][i + 1]].sum() for i in range(n)])
    return out
