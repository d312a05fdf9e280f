import numpy as np
def build(rp, ci, deg, SB=15, L=64, nctas=148, TR=1024, PMAX=6144):
    """block-SELL v3: p1 writes piece partials in stream order (block, row, piece); p2 stages each
    row tile's pieces (runs per block) into smem and sums each row's pieces via a local index."""
    n = len(rp) - 1; nnz = len(ci)
    order = np.argsort(-deg.astype(np.int64), kind='stable'); perm = np.empty(n, np.int64); perm[order] = np.arange(n)
    ncols = int((deg > 0).sum())
    g = perm[ci]
    lens = np.diff(rp); row = np.repeat(np.arange(n, dtype=np.int64), lens)
    b = g >> SB
    nb = int(b.max()) + 1 if nnz else 0
    key = b * (n + 1) + row
    idx = np.argsort(key, kind='stable')
    ks = key[idx]; bs = b[idx]
    bcnt = np.bincount(b, minlength=nb)
    SL = 32 * L
    nsl_b = (bcnt + SL - 1) // SL
    bstart = np.r_[0, np.cumsum(bcnt)][:-1]
    pstart = np.r_[0, np.cumsum(nsl_b * SL)][:-1]
    e = np.arange(nnz)
    ppos = pstart[bs] + (e - bstart[bs])
    chunk = ppos // L
    last_pair = np.r_[ks[1:] != ks[:-1], True]
    last_chunk = np.r_[chunk[1:] != chunk[:-1], True]
    flag = last_pair | last_chunk
    pend = np.flatnonzero(flag)
    npieces = len(pend)
    prow = ks[pend] % (n + 1); pblk = ks[pend] // (n + 1)
    nchunks = int((nsl_b * 32).sum())
    hdr = np.zeros(nchunks, np.int64)
    pfirst = np.r_[0, pend[:-1] + 1]
    cfirst = chunk[pfirst]
    uc, fi = np.unique(cfirst, return_index=True)
    hdr[uc] = fi
    k = ppos % L; s = chunk // 32; j = chunk % 32
    pos16 = ((s * (L // 8) + k // 8) * 32 + j) * 8 + k % 8
    lcol = np.zeros(nchunks * L, np.uint16)
    lcol[pos16] = ((g[idx] & ((1 << SB) - 1)) | (flag.astype(np.int64) << 15)).astype(np.uint16)
    sblk = np.repeat(np.arange(nb), nsl_b).astype(np.int32)
    nslices = len(sblk)
    cs = np.round(np.linspace(0, nslices, nctas + 1)).astype(np.int32)
    # ---- p2 tiles
    rcnt = np.bincount(prow, minlength=n)
    rslot = np.r_[0, np.cumsum(rcnt)]
    tiles = [0]
    cum = np.r_[0, np.cumsum(rcnt)]
    r0 = 0
    while r0 < n:
        r1 = min(n, r0 + TR)
        # shrink so that pieces <= PMAX
        lim = np.searchsorted(cum, cum[r0] + PMAX, side='right') - 1
        r1 = max(r0 + 1, min(r1, lim))
        tiles.append(r1); r0 = r1
    tiles = np.array(tiles, np.int64); ntiles = len(tiles) - 1
    ptile = np.searchsorted(tiles, prow, side='right') - 1      # tile of each piece (stream order)
    # run starts: first stream index of pieces with (block b, tile t)
    tb = pblk * ntiles + ptile                                   # stream order is sorted by (block, row) => by (block, tile)
    starts = np.searchsorted(tb, np.arange(nb * ntiles + 1))     # [b * ntiles + t]
    runlen = np.diff(starts).reshape(nb, ntiles).T               # [t][b]
    rstart = starts[:-1].reshape(nb, ntiles).T                   # [t][b]
    pre = np.zeros((ntiles, nb + 1), np.int64); pre[:, 1:] = np.cumsum(runlen, axis=1)
    # local index of each piece
    loc = pre[ptile, pblk] + (np.arange(npieces) - rstart[ptile, pblk])
    # slot order (row, block, stream idx)
    so_ = np.lexsort((np.arange(npieces), pblk, prow))
    qidx = loc[so_].astype(np.uint16)
    assert pre[:, -1].max() <= PMAX
    gpos = np.where(deg > 0, perm, -1).astype(np.int32)
    return dict(n=n, ncols=ncols, SB=SB, L=L, nb=nb, nslices=nslices, sblk=sblk, cs=cs, hdr=hdr.astype(np.int32),
                lcol=lcol, rslot=rslot.astype(np.int32), gpos=gpos, nslots=npieces, perm=perm,
                ntiles=ntiles, tiles=tiles.astype(np.int32), rstart=rstart.astype(np.int32).ravel(), pre=pre.astype(np.int32).ravel(), qidx=qidx)

def emulate(p, y_g):
    L = p['L']; S = 1 << p['SB']; nb = p['nb']
    part = np.full(p['nslots'], np.nan)
    for s in range(p['nslices']):
        b = p['sblk'][s]
        for j in range(32):
            c = 32 * s + j; pi = p['hdr'][c]; acc = 0.0
            for k in range(L):
                e = int(p['lcol'][((s * (L // 8) + k // 8) * 32 + j) * 8 + k % 8])
                col = b * S + (e & 0x7fff)
                acc += float(y_g[col]) if col < len(y_g) else 0.0
                if e >> 15:
                    part[pi] = acc; pi += 1; acc = 0.0
    out = np.zeros(p['n'])
    for t in range(p['ntiles']):
        pre = p['pre'][t * (nb + 1):(t + 1) * (nb + 1)]; st = p['rstart'][t * nb:(t + 1) * nb]
        sm = np.zeros(pre[-1])
        for kk in range(pre[-1]):
            bb = np.searchsorted(pre, kk, side='right') - 1
            sm[kk] = part[st[bb] + kk - pre[bb]]
        for i in range(p['tiles'][t], p['tiles'][t + 1]):
            out[i] = sum(sm[p['qidx'][s]] for s in range(p['rslot'][i], p['rslot'][i + 1]))
    return out
