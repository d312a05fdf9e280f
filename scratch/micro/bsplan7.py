import numpy as np
def build(rp, ci, deg, S=32768, LMAX=128, nctas=148, TR=512, PMAX=3072):
    """v7: lane-per-piece SELL in (block, tile, -len) order; part written coalesced at SELL position;
    padding entries point at the sentinel smem slot S (value 0)."""
    n = len(rp) - 1; nnz = len(ci)
    order = np.argsort(-deg.astype(np.int64), kind='stable'); perm = np.empty(n, np.int64); perm[order] = np.arange(n)
    ncols = int((deg > 0).sum())
    g = perm[ci]
    lens = np.diff(rp); row = np.repeat(np.arange(n, dtype=np.int64), lens)
    b = g // S
    nb = int(b.max()) + 1 if nnz else 0
    key = b * (n + 1) + row
    idx = np.argsort(key, kind='stable')
    ks = key[idx]
    brk = np.flatnonzero(np.r_[True, ks[1:] != ks[:-1]])
    pcnt = np.diff(np.r_[brk, nnz]); pst = brk
    pblk = ks[brk] // (n + 1); prow = ks[brk] % (n + 1)
    nsub = (pcnt + LMAX - 1) // LMAX
    sp = np.repeat(np.arange(len(pcnt)), nsub)
    sk = np.arange(len(sp)) - np.repeat(np.cumsum(nsub) - nsub, nsub)
    qst = pst[sp] + sk * LMAX; qlen = np.minimum(LMAX, pcnt[sp] - sk * LMAX)
    qblk = pblk[sp]; qrow = prow[sp]
    npieces = len(qst)
    # slots: (row, block, sub) order == current order sorted by row (stable)
    rcnt = np.bincount(qrow, minlength=n); rslot = np.r_[0, np.cumsum(rcnt)]
    cum = rslot
    tiles = [0]; r0 = 0
    while r0 < n:
        lim = np.searchsorted(cum, cum[r0] + PMAX, side='right') - 1
        r1 = max(r0 + 1, min(r0 + TR, lim)); tiles.append(r1); r0 = r1
    tiles = np.array(tiles, np.int64); ntiles = len(tiles) - 1
    qtile = np.searchsorted(tiles, qrow, side='right') - 1
    # SELL order: (block, tile, -len, row, sub)
    sel = np.lexsort((sk, qrow, -qlen, qtile, qblk))
    # pad each block to a multiple of 32
    bc = np.bincount(qblk, minlength=nb); nq_b = (bc + 31) // 32
    padb = np.r_[0, np.cumsum(nq_b * 32 - bc)][:-1]
    pos = np.arange(npieces) + np.repeat(padb, bc)      # SELL position of sel[i]
    tot = int((nq_b * 32).sum()); nslices = tot // 32
    L = np.zeros(tot, np.int64); L[pos] = qlen[sel]
    Ls = L.reshape(nslices, 32).max(1)
    soff = np.r_[0, np.cumsum(32 * Ls)][:-1]
    sblk = np.repeat(np.arange(nb), nq_b)
    # lcol [slice][k][lane], sentinel S for padding
    lcol = np.full(int(32 * Ls.sum()), S, np.int64)
    E = qlen[sel]
    lane_pos = np.repeat(pos, E)
    kk = np.arange(int(E.sum())) - np.repeat(np.cumsum(E) - E, E)
    src = idx[np.repeat(qst[sel], E) + kk]
    sl = lane_pos // 32; ln = lane_pos % 32
    lcol[soff[sl] + 32 * kk + ln] = g[src] - sblk[sl] * S
    assert lcol.max() <= S and S < 65536
    # run table per (tile, block): range of SELL positions
    spos = np.empty(npieces, np.int64); spos[sel] = pos           # SELL position of piece q
    tb = qblk * ntiles + qtile
    # runs: pieces with same (block, tile) are contiguous in SELL order
    order_tb = np.argsort(spos)
    tbs = tb[order_tb]; ps = spos[order_tb]
    starts = np.searchsorted(tbs, np.arange(nb * ntiles + 1))
    rstart_pos = np.where(starts[:-1] < npieces, ps[np.minimum(starts[:-1], npieces - 1)], 0)
    runlen = np.diff(starts)
    rs = rstart_pos.reshape(nb, ntiles).T; rl = runlen.reshape(nb, ntiles).T
    pre = np.zeros((ntiles, nb + 1), np.int64); pre[:, 1:] = np.cumsum(rl, axis=1)
    loc = pre[qtile, qblk] + (spos - rs[qtile, qblk])
    so_ = np.lexsort((sk, qblk, qrow))           # slot order (row, block, sub)
    qidx = loc[so_].astype(np.uint16)
    # CTA partition of slices by entries (block-major), warps split inside
    w = 32 * Ls + 32
    cw = np.r_[0, np.cumsum(w)]
    cs = np.searchsorted(cw, np.linspace(0, cw[-1], nctas + 1), side='left').astype(np.int32); cs[-1] = nslices
    gpos = np.where(deg > 0, perm, -1).astype(np.int32)
    tinfo = np.stack([tiles[:-1], tiles[1:], rslot[tiles[:-1]], rslot[tiles[1:]]], 1).astype(np.int32)
    # run table interleaved (start, len) per (tile, block)
    runs = np.stack([rs, rl], 2).astype(np.int32)
    return dict(n=n, ncols=ncols, S=S, nb=nb, nslices=nslices, sblk=sblk.astype(np.int32), soff=soff.astype(np.int32),
                sL=Ls.astype(np.int32), cs=cs, lcol=lcol.astype(np.uint16), rslot=rslot.astype(np.int32), gpos=gpos, npieces=npieces,
                perm=perm, ntiles=ntiles, tinfo=np.ascontiguousarray(tinfo), runs=np.ascontiguousarray(runs.reshape(-1)), pre=pre.astype(np.int32).ravel(), qidx=qidx,
                nslots_sell=tot)

def emulate(p, y_g):
    S = p['S']; nb = p['nb']
    part = np.zeros(p['nslots_sell'])
    for s in range(p['nslices']):
        b = p['sblk'][s]; L = p['sL'][s]; off = p['soff'][s]
        xs = np.zeros(S + 1); cn = min(S, len(y_g) - b * S); xs[:cn] = y_g[b * S: b * S + cn]
        blk = p['lcol'][off: off + 32 * L].reshape(L, 32).astype(np.int64)
        part[32 * s: 32 * s + 32] = xs[blk].sum(0)
    out = np.zeros(p['n'])
    for t in range(p['ntiles']):
        R0, R1, S0, S1 = p['tinfo'][t]
        runs = p['runs'][t * nb * 2:(t + 1) * nb * 2].reshape(nb, 2)
        sm = np.concatenate([part[st: st + ln] for st, ln in runs])
        for i in range(R0, R1):
            out[i] = sum(sm[p['qidx'][s]] for s in range(p['rslot'][i], p['rslot'][i + 1]))
    return out
