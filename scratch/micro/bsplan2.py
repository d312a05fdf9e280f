import numpy as np
def build(rp, ci, deg, SB=15, L=64, nctas=148):
    """block-SELL v2: per block, entries in (row, position) order cut into lane chunks of L entries;
    pieces = pairs (row, block) cut at chunk boundaries; last entry of each piece flagged (bit 15)."""
    n = len(rp) - 1; nnz = len(ci)
    order = np.argsort(-deg.astype(np.int64), kind='stable'); perm = np.empty(n, np.int64); perm[order] = np.arange(n)
    ncols = int((deg > 0).sum())
    g = perm[ci]
    lens = np.diff(rp); row = np.repeat(np.arange(n, dtype=np.int64), lens)
    b = g >> SB
    nb = int(b.max()) + 1 if nnz else 0
    key = b * (n + 1) + row
    idx = np.argsort(key, kind='stable')             # entries by (block, row, position)
    ks = key[idx]; bs = b[idx]
    # per block: entries padded to a multiple of 32L (one slice = 32 lane chunks of L)
    bcnt = np.bincount(b, minlength=nb)
    SL = 32 * L
    nsl_b = (bcnt + SL - 1) // SL
    bstart = np.r_[0, np.cumsum(bcnt)][:-1]
    pstart = np.r_[0, np.cumsum(nsl_b * SL)][:-1]
    # position of each sorted entry in the padded stream
    e = np.arange(nnz)
    ppos = pstart[bs] + (e - bstart[bs])                # padded linear position
    chunk = ppos // L
    # piece end: last entry of a pair, or last entry of a chunk
    last_pair = np.r_[ks[1:] != ks[:-1], True]
    last_chunk = np.r_[chunk[1:] != chunk[:-1], True]
    flag = last_pair | last_chunk
    # pieces in stream order
    pend = np.flatnonzero(flag)
    npieces = len(pend)
    prow = ks[pend] % (n + 1); pblk = ks[pend] // (n + 1)
    # piece order within a pair -> slot order (row, block, piece)
    so_ = np.lexsort((np.arange(npieces), pblk, prow))
    slot = np.empty(npieces, np.int64); slot[so_] = np.arange(npieces)
    rslot = np.zeros(n + 1, np.int64); np.add.at(rslot, prow + 1, 1); rslot = np.cumsum(rslot)
    # lane headers: index of first piece of each chunk
    nchunks = int((nsl_b * 32).sum())
    hdr = np.zeros(nchunks, np.int64)
    pstart_piece = np.r_[0, pend[:-1] + 1]           # first entry (sorted idx) of each piece
    cfirst = chunk[pstart_piece]
    # first piece of chunk c = min piece index whose first entry is in chunk c
    uc, fi = np.unique(cfirst, return_index=True)
    hdr[uc] = fi
    # SELL-interleaved lcol: chunk c = (slice s, lane j) with s = c // 32, j = c % 32; entry k of chunk:
    # u16 index = ((s * (L/8) + k // 8) * 32 + j) * 8 + k % 8
    k = ppos % L; s = chunk // 32; j = chunk % 32
    pos16 = ((s * (L // 8) + k // 8) * 32 + j) * 8 + k % 8
    lcol = np.zeros(nchunks * L, np.uint16)
    lcol[pos16] = ((g[idx] & ((1 << SB) - 1)) | (flag.astype(np.int64) << 15)).astype(np.uint16)
    sblk = np.repeat(np.arange(nb), nsl_b).astype(np.int32)
    nslices = len(sblk)
    cs = np.round(np.linspace(0, nslices, nctas + 1)).astype(np.int32)
    gpos = np.where(deg > 0, perm, -1).astype(np.int32)
    return dict(n=n, ncols=ncols, SB=SB, L=L, nslices=nslices, sblk=sblk, cs=cs, hdr=hdr.astype(np.int32),
                pslot=slot.astype(np.int32), lcol=lcol, rslot=rslot.astype(np.int32), gpos=gpos, nslots=npieces, perm=perm)

def emulate(p, y_g):
    L = p['L']; S = 1 << p['SB']
    part = np.full(p['nslots'], np.nan)
    for s in range(p['nslices']):
        b = p['sblk'][s]
        for j in range(32):
            c = 32 * s + j; pi = p['hdr'][c]; acc = 0.0
            for k in range(L):
                e = int(p['lcol'][((s * (L // 8) + k // 8) * 32 + j) * 8 + k % 8])
                acc += float(y_g[b * S + (e & 0x7fff)]) if b * S + (e & 0x7fff) < len(y_g) else 0.0
                if e >> 15:
                    part[p['pslot'][pi]] = acc; pi += 1; acc = 0.0
    n = p['n']
    return np.array([part[p['rslot'][i]:p['rslot'][i + 1]].sum() for i in range(n)])
