# 2D-staged SpMV plan v5 (design study, numpy): warm columns (< CUT) staged per tile (v4 layout),
# cold columns gathered from L2 in a per-panel cold phase (pieces / slices with u32 indices).  Row panels x column tiles of the gather layout.
#
# Panel  = contiguous rows (multiples of 32), cost-balanced, <= NRMAX non-empty rows (fp64
#          accumulators in shared memory, compact index = rank among the panel's non-empty rows).
# Hot    = columns [0, H) of the gather layout, resident in shared memory for the whole launch.
# Tile   = (panel, column range): <= SMAX distinct 32-byte cold sectors of x (staged into shared
#          memory, compacted: slot k holds sector secs[k]) and <= WMAX work (2 x entries).
# Entry  = u16 index into one shared array [stage0 | 8 zeros | hot | stage1 | 8 zeros] from the tile's
#          base: even tiles (inside the panel) use base 0: staged slot*8 + (g&7), zero S8, hot S8+8+g;
#          odd tiles base S8+8: hot g, staged H + slot*8 + (g&7), zero H+S8  (S8 = SMAX*8).
# Pairs  = the entries of one row in one tile (row order kept: position order inside a tile).
#          long (>= LTH): pieces of <= PIECE entries, lane-strided 8-entry groups + xor tree;
#          short: slices of 32 pairs sorted by length, one lane per pair, [k][lane] layout.
import numpy as np



def build(rp, ci, NRMAX=8192, WMAX=12288, LTH=32, PIECE=512, ROWW=2, BLOBMAX=16384, H=0, SMAX=768, G=148, CUT=262144, CLTH=32):
    n = rp.shape[0] - 1
    nnz = ci.shape[0]
    cnt = np.bincount(ci, minlength=n)
    order = np.argsort(-cnt, kind='stable')
    newid = np.empty(n, np.int64)
    newid[order] = np.arange(n)
    ncols_g = int((cnt > 0).sum())
    g = newid[ci]
    rowlen = np.diff(rp)
    ne = rowlen > 0
    # ---------------- panels (cuts at multiples of 32 rows)
    ngr = (n + 31) // 32
    pad = ngr * 32 - n
    rl = np.concatenate([rowlen, np.zeros(pad, np.int64)])
    nel = np.concatenate([ne, np.zeros(pad, bool)])
    gcost = (rl + ROWW).reshape(ngr, 32).sum(1)
    gnr = nel.reshape(ngr, 32).sum(1)
    cc = np.concatenate([[0], np.cumsum(gcost)])
    cn = np.concatenate([[0], np.cumsum(gnr)])
    total = cc[-1]
    # G cost-balanced row ranges (one per CTA), each cut into sub-panels of <= NRMAX non-empty rows
    cuts = [0]
    ccut = np.searchsorted(cc, np.linspace(0, total, G + 1)[1:-1], 'left')
    bnd = np.concatenate([[0], np.maximum.accumulate(np.clip(ccut, 0, ngr)), [ngr]])
    cta_of_pan = []
    for b_ in range(G):
        s0, s1 = int(bnd[b_]), int(bnd[b_ + 1])
        nrr = cn[s1] - cn[s0]
        k_ = max(1, int(-(-nrr // NRMAX)))
        while True:
            sub = np.searchsorted(cn, cn[s0] + np.arange(1, k_) * nrr / k_, 'left')
            sc = [s0] + [int(v) for v in np.clip(sub, s0, s1)] + [s1]
            if all(cn[sc[i + 1]] - cn[sc[i]] <= NRMAX for i in range(k_)):
                break
            k_ += 1
        for i in range(k_):
            if sc[i + 1] > sc[i]:
                cuts.append(sc[i + 1]); cta_of_pan.append(b_)
    cuts = np.array(cuts, np.int64)
    cta_of_pan = np.array(cta_of_pan, np.int64)
    assert cuts.shape[0] == cta_of_pan.shape[0] + 1
    npan = cuts.shape[0] - 1
    pan_of_grp = np.repeat(np.arange(npan), np.diff(cuts))
    pan_of_row = pan_of_grp[np.arange(n) >> 5]
    # compact accumulator index of each non-empty row inside its panel
    cne = np.cumsum(ne) - ne                       # non-empty rows before row i (global)
    first_row = cuts[:-1] * 32
    rloc = cne - cne[np.minimum(first_row, n - 1)][pan_of_row]
    grp_mask = np.packbits(nel.reshape(ngr, 32)[:, ::-1], axis=1, bitorder='big').view('>u4').astype(np.uint32).reshape(ngr)
    gbase = (cn[:-1] - cn[cuts[:-1]][pan_of_grp]).astype(np.int32)
    # ---------------- tiles: per panel, the gather-layout column axis is cut into ranges (no
    # sector is staged twice inside a panel): hot range [0, H) (resident cache, no staging) cut by
    # work only, the rest cut by work (2 x entries, an upper bound of entries + pairs) and sectors.
    row_all = np.repeat(np.arange(n, dtype=np.int64), rowlen)
    warm_e = g < CUT
    cold_e = np.nonzero(~warm_e)[0]
    g_all = g
    row = row_all[warm_e]
    g = g[warm_e]
    epan = pan_of_row[row]
    sec = g >> 3
    hot = g < H
    skey = epan * (1 << 27) + sec
    us, scnt = np.unique(skey, return_counts=True)
    s_pan = us >> 27
    s_sec = us & ((1 << 27) - 1)
    s_hot = s_sec < (H >> 3)
    s_first = np.searchsorted(s_pan, np.arange(npan))
    s_end = np.concatenate([s_first[1:], [us.shape[0]]])
    tile_of_s = np.empty(us.shape[0], np.int64)
    tile_pan = []
    t = -1
    for p in range(npan):
        a_, b_ = int(s_first[p]), int(s_end[p])
        if a_ == b_:
            continue
        w = np.cumsum(2 * scnt[a_:b_])
        hcount = int(s_hot[a_:b_].sum())
        st = 0
        m = b_ - a_
        while st < m:
            base = w[st - 1] if st > 0 else 0
            en = int(np.searchsorted(w, base + WMAX, 'right'))
            if st < hcount:
                en = min(en, hcount)
            else:
                en = min(en, st + SMAX)
            en = max(en, st + 1)
            t += 1
            tile_pan.append(p)
            tile_of_s[a_ + st:a_ + en] = t
            st = en
    ntile = t + 1
    tile_pan = np.array(tile_pan, np.int64)
    etile = tile_of_s[np.searchsorted(us, skey)]
    # staged sectors per tile (cold only), slot = rank inside the tile
    t_first_s = np.searchsorted(tile_of_s, np.arange(ntile))
    cold_s = ~s_hot
    cs_cold = np.concatenate([[0], np.cumsum(cold_s)])
    tfirst = cs_cold[t_first_s]
    tnsec = np.diff(np.concatenate([tfirst, [cs_cold[-1]]]))
    tsec = s_sec[cold_s]
    assert tnsec.max() <= SMAX, tnsec.max()
    sidx = np.searchsorted(us, skey)
    slot = cs_cold[sidx] - tfirst[etile]
    S8 = SMAX * 8
    tpar = (np.arange(ntile) - np.searchsorted(tile_pan, tile_pan)) & 1      # tile index inside its panel, mod 2
    epar = tpar[etile]
    assert H == 0
    local = (slot * 8 + (g & 7)).astype(np.uint16)
    # entries in (tile, row, position) order: stable by tile keeps CSR order
    eo = np.argsort(etile, kind='stable')
    loc_s = local[eo]
    row_s = row[eo]
    tile_s = etile[eo]
    # pairs in tile order
    tp_key = tile_s * n + row_s
    pk2, pst2, pc2 = np.unique(tp_key, return_index=True, return_counts=True)
    p_tile = pk2 // n
    p_row = pk2 % n
    p_first = np.searchsorted(p_tile, np.arange(ntile))
    p_end = np.concatenate([p_first[1:], [pk2.shape[0]]])
    # ---------------- blobs: per tile [items (4 u16 each, LPT order)] [combines (4 u16)] [slice slot lists] [entries]
    # piece  {off8, l8, slot, 0xFFFF}           direct: ACC[slot] += lane-strided sum
    # sub    {off8, l8, cmb, pslot}             partial -> PART[pslot]; last of combine cmb sums them
    # slice  {off8, L | 0x8000, rows8, 0}       lane l: ACC[rows[l]] += sum of [k][lane] entries
    # combine{slot, pfirst, count, 0}
    rows_l = rloc[p_row].astype(np.int64)
    longm = pc2 >= LTH
    lj = np.nonzero(longm)[0]
    npc = (pc2[lj] + PIECE - 1) // PIECE
    pc_pair = np.repeat(lj, npc)
    pc_q = np.arange(pc_pair.shape[0]) - np.repeat(np.cumsum(npc) - npc, npc)
    pc_len = np.minimum(PIECE, pc2[pc_pair] - pc_q * PIECE)
    pc_l8 = (pc_len + 7) // 8
    pc_tile = p_tile[pc_pair]
    pc_direct = np.repeat(npc == 1, npc)
    multi = ~pc_direct
    tmfirst = np.searchsorted(pc_tile, np.arange(ntile))
    mcs = np.cumsum(multi) - multi
    mbase = np.concatenate([mcs, [int(multi.sum())]])[tmfirst]
    pc_pslot = np.where(pc_direct, 0xFFFF, mcs - mbase[pc_tile])
    cj = lj[npc > 1]
    cb_tile = p_tile[cj]
    cfirst_t = np.searchsorted(cb_tile, np.arange(ntile))
    cb_idx = np.arange(cj.shape[0]) - cfirst_t[cb_tile]
    pc_cmb = np.where(pc_direct, 0, np.repeat(np.where(npc > 1, 0, 0), npc))
    # combine id of each sub-piece
    cmb_of_pair = np.full(pc2.shape[0], -1, np.int64)
    cmb_of_pair[cj] = cb_idx
    pc_cmb = np.where(pc_direct, rows_l[pc_pair], cmb_of_pair[pc_pair])
    cb_first = pc_pslot[np.searchsorted(pc_pair, cj)]
    cb_n = npc[npc > 1]
    # short pairs -> CTA-wide slices sorted by (tile, -len)
    sj = np.nonzero(~longm)[0]
    so = np.lexsort((-pc2[sj], p_tile[sj]))
    sj = sj[so]
    s_tile = p_tile[sj]
    sfirst = np.searchsorted(s_tile, np.arange(ntile))
    srank = np.arange(sj.shape[0]) - sfirst[s_tile]
    s_lane = srank % 32
    s_sl_local = srank // 32
    nsl_t = np.zeros(ntile, np.int64)
    np.maximum.at(nsl_t, s_tile, s_sl_local + 1)
    slbase = np.concatenate([[0], np.cumsum(nsl_t)])
    s_sl = slbase[s_tile] + s_sl_local
    nslices = int(slbase[-1])
    sl_L = np.zeros(nslices, np.int64)
    np.maximum.at(sl_L, s_sl, pc2[sj])
    sl_tile = np.repeat(np.arange(ntile), nsl_t)
    np_t = np.bincount(pc_tile, minlength=ntile)
    nc_t = np.bincount(cb_tile, minlength=ntile)
    ni_t = np_t + nsl_t
    hdr = 4 * ni_t + 4 * nc_t + 32 * nsl_t
    hdr = (hdr + 7) // 8 * 8
    pe_t = np.bincount(pc_tile, weights=pc_l8 * 8, minlength=ntile).astype(np.int64)
    se_t = np.bincount(sl_tile, weights=sl_L * 32, minlength=ntile).astype(np.int64)
    tot_t = hdr + pe_t + se_t
    assert (tot_t * 2).max() <= BLOBMAX, (tot_t * 2).max()
    toff = np.concatenate([[0], np.cumsum(tot_t)])
    blob = np.full(int(toff[-1]), S8, np.uint16)
    ent0 = toff[:-1] + hdr
    # entry offsets (absolute u16): pieces first, then slices
    pcs = np.cumsum(pc_l8 * 8) - pc_l8 * 8
    pcs_s = np.concatenate([pcs, [0]])
    p_abs = ent0[pc_tile] + pcs - pcs_s[tmfirst][pc_tile]
    slfirst = np.searchsorted(sl_tile, np.arange(ntile))
    scs = np.cumsum(sl_L * 32) - sl_L * 32
    scs_s = np.concatenate([scs, [0]])
    s_abs = ent0[sl_tile] + pe_t[sl_tile] + scs - scs_s[slfirst][sl_tile]
    # items in LPT order per tile: cost = entries (pieces l8*8, slices L*32)
    it_tile = np.concatenate([pc_tile, sl_tile])
    it_cost = np.concatenate([pc_l8 * 8, sl_L * 32])
    it_kind = np.concatenate([np.zeros(pc_tile.shape[0], np.int64), np.ones(nslices, np.int64)])
    it_id = np.concatenate([np.arange(pc_tile.shape[0]), np.arange(nslices)])
    io = np.lexsort((-it_cost, it_tile))
    it_tile, it_kind, it_id = it_tile[io], it_kind[io], it_id[io]
    ifirst = np.searchsorted(it_tile, np.arange(ntile))
    it_rank = np.arange(io.shape[0]) - ifirst[it_tile]
    ib = toff[:-1][it_tile] + 4 * it_rank
    pk = it_kind == 0
    pid = it_id[pk]
    blob[ib[pk]] = (p_abs[pid] - toff[:-1][pc_tile[pid]]) // 8
    blob[ib[pk] + 1] = pc_l8[pid]
    blob[ib[pk] + 2] = pc_cmb[pid]
    blob[ib[pk] + 3] = pc_pslot[pid]
    sk = ~pk
    sid = it_id[sk]
    rows_rel = 4 * ni_t + 4 * nc_t                                  # u16 offset of the slot lists in the blob
    blob[ib[sk]] = (s_abs[sid] - toff[:-1][sl_tile[sid]]) // 8
    blob[ib[sk] + 1] = sl_L[sid] | 0x8000
    sidx = np.arange(nslices) - slfirst[sl_tile]
    rl_off = rows_rel[sl_tile] + 32 * sidx                          # multiple of 8? rows_rel is 4*(ni+nc)
    blob[ib[sk] + 2] = rl_off[sid]
    blob[ib[sk] + 3] = 0
    for l in range(32):
        blob[toff[:-1][sl_tile] + rl_off + l] = 0xFFFF
    blob[toff[:-1][s_tile] + rl_off[s_sl] + s_lane] = rows_l[sj]
    # combines
    hb = toff[:-1][cb_tile] + 4 * ni_t[cb_tile] + 4 * cb_idx
    blob[hb] = rows_l[cj]
    blob[hb + 1] = cb_first
    blob[hb + 2] = cb_n
    blob[hb + 3] = 0
    # entries
    tot_pe = int(pc_len.sum())
    rp_ = np.repeat(np.arange(pc_pair.shape[0]), pc_len)
    kk = np.arange(tot_pe) - np.repeat(np.cumsum(pc_len) - pc_len, pc_len)
    blob[p_abs[rp_] + kk] = loc_s[pst2[pc_pair][rp_] + pc_q[rp_] * PIECE + kk]
    L_s = pc2[sj]
    rs_ = np.repeat(np.arange(sj.shape[0]), L_s)
    kk = np.arange(rs_.shape[0]) - np.repeat(np.cumsum(L_s) - L_s, L_s)
    blob[s_abs[s_sl][rs_] + kk * 32 + s_lane[rs_]] = loc_s[pst2[sj][rs_] + kk]
    stats = dict(pieces=int(pc_pair.shape[0]), slices=nslices, combines=int(cj.shape[0]),
                 padded=int((pe_t + se_t).sum()), blobmax=int((tot_t * 2).max()),
                 pmax=int(np.bincount(pc_tile[multi], minlength=ntile).max()) if multi.any() else 0,
                 cmax=int(nc_t.max()), imax=int(ni_t.max()))
    blobs = blob
    # panels: {grp_begin, grp_end, tile_begin, tile_end, nr}
    tb = np.searchsorted(tile_pan, np.arange(npan))
    te = np.concatenate([tb[1:], [ntile]])
    nr = (cn[cuts[1:]] - cn[cuts[:-1]])
    prec_ = np.stack([cuts[:-1], cuts[1:], tb, te, nr, np.zeros(npan, np.int64), np.zeros(npan, np.int64),
                      np.zeros(npan, np.int64)], 1).astype(np.int32)
    # ---------------- cold part (columns >= CUT): per panel, one pair per row with cold entries
    # (position order), gathered straight from L2 by the cold phase after the panel's warm tiles.
    # citems int4: piece {off, len, slot|cmb, -1|pslot}; slice {off, L | 1<<30, rows_off, 0}
    # cidx: u32 gather-layout indices (pieces contiguous, 4-aligned; slices [k][lane]); ZIDX pads
    ZIDX = ncols_g
    c_row = row_all[cold_e]
    c_pan = pan_of_row[c_row]
    c_g = g_all[cold_e]
    cu, cst, clen = np.unique(c_row, return_index=True, return_counts=True)
    cpan = pan_of_row[cu]
    crl = rloc[cu]
    clong = clen >= CLTH
    lj = np.nonzero(clong)[0]
    npc = (clen[lj] + PIECE - 1) // PIECE
    pp = np.repeat(lj, npc)
    pq = np.arange(pp.shape[0]) - np.repeat(np.cumsum(npc) - npc, npc)
    plen = np.minimum(PIECE, clen[pp] - pq * PIECE)
    pdirect = np.repeat(npc == 1, npc)
    ppan = cpan[pp]
    # partial slots and combines per panel
    multi = ~pdirect
    pfirst_p = np.searchsorted(ppan, np.arange(npan))
    mcs = np.cumsum(multi) - multi
    mb = np.concatenate([mcs, [int(multi.sum())]])[pfirst_p]
    ppslot = np.where(pdirect, -1, mcs - mb[ppan])
    cj = lj[npc > 1]
    cjpan = cpan[cj]
    cfirst_p = np.searchsorted(cjpan, np.arange(npan))
    cidx_in_pan = np.arange(cj.shape[0]) - cfirst_p[cjpan]
    cmb_of = np.full(cu.shape[0], -1, np.int64)
    cmb_of[cj] = cidx_in_pan
    pa = np.where(pdirect, crl[pp], cmb_of[pp])
    ccomb = np.zeros((cj.shape[0], 4), np.int64)
    ccomb[:, 0] = crl[cj]
    ccomb[:, 1] = ppslot[np.searchsorted(pp, cj)]
    ccomb[:, 2] = npc[npc > 1]
    # short cold pairs: slices of 32 per panel, sorted by length desc
    sj = np.nonzero(~clong)[0]
    sj = sj[np.lexsort((-clen[sj], cpan[sj]))]
    spn = cpan[sj]
    sfp = np.searchsorted(spn, np.arange(npan))
    srk = np.arange(sj.shape[0]) - sfp[spn]
    sln = srk % 32
    ssl_loc = srk // 32
    nsl_p = np.zeros(npan, np.int64)
    np.maximum.at(nsl_p, spn, ssl_loc + 1)
    slb = np.concatenate([[0], np.cumsum(nsl_p)])
    ssl = slb[spn] + ssl_loc
    nsl = int(slb[-1])
    slL = np.zeros(nsl, np.int64)
    np.maximum.at(slL, ssl, clen[sj])
    sl_pan = np.repeat(np.arange(npan), nsl_p)
    # index array layout: per panel, pieces (4-aligned) then slices
    p4 = (plen + 3) // 4 * 4
    psz_p = np.bincount(ppan, weights=p4, minlength=npan).astype(np.int64)
    ssz_p = np.bincount(sl_pan, weights=slL * 32, minlength=npan).astype(np.int64)
    pbase = np.concatenate([[0], np.cumsum(psz_p + ssz_p)])
    cidx = np.full(int(pbase[-1]), ZIDX, np.int64)
    pcs = np.cumsum(p4) - p4
    pcs_s = np.concatenate([pcs, [0]])
    poff = pbase[:-1][ppan] + pcs - pcs_s[pfirst_p][ppan]
    rr = np.repeat(np.arange(pp.shape[0]), plen)
    kk = np.arange(rr.shape[0]) - np.repeat(np.cumsum(plen) - plen, plen)
    cidx[poff[rr] + kk] = c_g[cst[pp][rr] + pq[rr] * PIECE + kk]
    slfp = np.searchsorted(sl_pan, np.arange(npan))
    scs = np.cumsum(slL * 32) - slL * 32
    scs_s = np.concatenate([scs, [0]])
    soff = pbase[:-1][sl_pan] + psz_p[sl_pan] + scs - scs_s[slfp][sl_pan]
    L_ = clen[sj]
    rr = np.repeat(np.arange(sj.shape[0]), L_)
    kk = np.arange(rr.shape[0]) - np.repeat(np.cumsum(L_) - L_, L_)
    cidx[soff[ssl][rr] + kk * 32 + sln[rr]] = c_g[cst[sj][rr] + kk]
    crows = np.full(nsl * 32, 0xFFFF, np.int64)
    crows[ssl * 32 + sln] = crl[sj]
    # items per panel in LPT order
    it_pan = np.concatenate([ppan, sl_pan])
    it_cost = np.concatenate([plen, slL * 32])
    rec = np.zeros((it_pan.shape[0], 4), np.int64)
    rec[:pp.shape[0], 0] = poff
    rec[:pp.shape[0], 1] = plen
    rec[:pp.shape[0], 2] = pa
    rec[:pp.shape[0], 3] = ppslot
    rec[pp.shape[0]:, 0] = soff
    rec[pp.shape[0]:, 1] = slL | (1 << 30)
    rec[pp.shape[0]:, 2] = np.arange(nsl) * 32
    io = np.lexsort((-it_cost, it_pan))
    citems = rec[io]
    ci_first = np.searchsorted(it_pan[io], np.arange(npan + 1))
    cc_first = np.searchsorted(cjpan, np.arange(npan + 1))
    cstats = dict(cold_entries=int(cold_e.shape[0]), cold_pieces=int(pp.shape[0]), cold_slices=nsl,
                  cold_idx=int(cidx.shape[0]), cold_pmax=int(np.bincount(ppan[multi], minlength=npan).max()) if multi.any() else 0,
                  cold_cmax=int(np.bincount(cjpan, minlength=npan).max()) if cj.shape[0] else 0)
    # per-CTA tile sequences (static round-robin of panels; a panel without tiles gets a null tile)
    trec = np.stack([toff[:-1] // 8, tot_t // 8, tfirst, tnsec, ni_t, nc_t, ni_t, np.zeros(ntile, np.int64)], 1).astype(np.int64)
    trec[:, 6] = 4 * ni_t            # u16 offset of the combine table
    trec[:, 7] = tile_pan
    seq = []
    seq_off = [0]
    flags = []
    for b_ in range(G):
        for p in np.nonzero(cta_of_pan == b_)[0]:
            for t_ in range(int(tb[p]), int(te[p])):
                seq.append(t_)
                flags.append(int(p))
            seq.append(-2 - int(p))          # cold phase + epilogue
            flags.append(int(p) | (1 << 30) | (1 << 29))
        seq_off.append(len(seq))
    seq = np.array(seq, np.int64)
    flags = np.array(flags, np.int64)
    seqrec = np.zeros((seq.shape[0], 8), np.int64)
    real = seq >= 0
    seqrec[real, :6] = trec[seq[real]][:, [0, 1, 2, 3, 4, 6]]
    cp_ = -2 - seq[~real]
    seqrec[~real, 0] = ci_first[cp_]
    seqrec[~real, 2] = cc_first[cp_]
    seqrec[~real, 4] = ci_first[cp_ + 1] - ci_first[cp_]
    seqrec[~real, 5] = cc_first[cp_ + 1] - cc_first[cp_]
    seqrec[:, 6] = flags
    seqrec[:, 7] = np.where(real, seq, -2)
    stats.update(npan=npan, ntile=ntile, sectors=int(tsec.shape[0]), pairs=int(pk2.shape[0]), nnz=nnz,
                 blob_bytes=int(blobs.shape[0] * 2), ncols_g=ncols_g, nrmax=int(nr.max()), H=H, SMAX=SMAX, G=G)
    perm = np.where(cnt > 0, newid, -1).astype(np.int32)
    stats.update(cstats)
    return dict(citems=citems.astype(np.int32), ccomb=ccomb.astype(np.int32), cidx=cidx.astype(np.uint32), crows=crows.astype(np.uint16), zidx=ZIDX, seqrec=seqrec.astype(np.int32), maxseq=int(np.diff(seq_off).max()), seq=seq.astype(np.int32), seqflags=flags.astype(np.int32), seqoff=np.array(seq_off, np.int32), pair_tile=p_tile, pair_row=p_row, pair_len=pc2, tile_pan=tile_pan, panels=prec_, tiles=trec.astype(np.int32), secs=tsec.astype(np.int32), blob=blobs, gmask=grp_mask, gbase=gbase,
                perm=perm, newid=newid, g=g_all, row=row_all, ncols_g=ncols_g, stats=stats)
