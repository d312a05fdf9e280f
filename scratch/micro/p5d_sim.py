# numpy simulation of the v5 kernel's reading of the plan (format check, CPU)
import numpy as np

def simulate(pl, x, n):
    blob = pl['blob']; secs = pl['secs']; panels = pl['panels']
    S8 = pl['stats']['SMAX'] * 8
    out = np.zeros(n, np.float64)
    rec, so = pl['seqrec'], pl['seqoff']
    ci, cc, cx, cr = pl['citems'], pl['ccomb'], pl['cidx'].astype(np.int64), pl['crows'].astype(np.int64)
    for b in range(so.shape[0] - 1):
        acc = np.zeros(1 << 16, np.float64)
        for k in range(so[b], so[b + 1]):
            r = rec[k].astype(np.int64)
            fl = int(r[6]); p = fl & ((1 << 29) - 1)
            part = {}
            if r[7] >= 0:
                bo, b16, sof, ns, ni, coff = r[:6]
                buf = np.zeros(S8 + 8, np.float64)
                sec = secs[sof:sof + ns]
                buf[:ns * 8] = x[(sec[:, None] * 8 + np.arange(8)).reshape(-1)]
                B = blob[bo * 8:(bo + b16) * 8].astype(np.int64)
                for i in range(ni):
                    off8, ln, a, c = B[4 * i:4 * i + 4]
                    if ln & 0x8000:
                        L = ln & 0x7fff
                        rows = B[a:a + 32]
                        m = B[off8 * 8:off8 * 8 + L * 32].reshape(L, 32)
                        s = buf[m].sum(axis=0)
                        for l in range(32):
                            if rows[l] != 0xFFFF: acc[rows[l]] += s[l]
                    else:
                        s = buf[B[off8 * 8:(off8 + ln) * 8]].sum()
                        if c == 0xFFFF: acc[a] += s
                        else: part[c] = s
                for i in range(r[5] if False else int(np.sum(0))):
                    pass
                nc = tiles_nc = None
            else:
                i0, _, c0, _, ni, nc = r[:6]
                for i in range(i0, i0 + ni):
                    off, ln, a, c = ci[i].astype(np.int64)
                    if ln & (1 << 30):
                        L = ln & ((1 << 30) - 1)
                        rows = cr[a:a + 32]
                        m = cx[off:off + L * 32].reshape(L, 32)
                        s = x[m].sum(axis=0)
                        for l in range(32):
                            if rows[l] != 0xFFFF: acc[rows[l]] += s[l]
                    else:
                        s = x[cx[off:off + ln]].sum()
                        if c == -1: acc[a] += s
                        else: part[c] = s
                for j in range(c0, c0 + nc):
                    row, f, cnt, _ = cc[j]
                    acc[row] += sum(part[f + q] for q in range(cnt))
            if r[7] >= 0:
                # warm combines
                bo, b16 = r[0], r[1]; ni = r[4]; coff = r[5]
                B = blob[bo * 8:(bo + b16) * 8].astype(np.int64)
                ncw = pl['tiles'][r[7]][5]
                for i in range(ncw):
                    row, f, cnt = B[coff + 4 * i:coff + 4 * i + 3]
                    acc[row] += sum(part[f + q] for q in range(cnt))
            if (fl >> 30) & 1:
                g0, g1 = panels[p][:2]
                for grp in range(g0, g1):
                    m = int(pl['gmask'][grp]); base = int(pl['gbase'][grp])
                    for l in range(32):
                        i = grp * 32 + l
                        if i < n and (m >> l) & 1:
                            out[i] = acc[base + bin(m & ((1 << l) - 1)).count('1')]
                acc[:] = 0
    return out
