"""Multi-GPU data plane on the CPU (world size 2, gloo) -- SURVEY 8(e), DESIGN.md section 8.

Each rank sweeps its row block of the symmetrically relabelled AT with the oracle's row kernel;
everything that decides WHERE data goes and HOW the scalars combine is the product's host code:
  * nbg_partition_rows        the byte-balanced cuts (the rule the GPU setup applies in pi-space),
  * nbg_dist_exchange_plan    each rank's slice of the gathered vector (clipped at ncols_g),
  * nbg_xacc_encode / decode  the exact-accumulator slot of the delta and the dangling mass,
and the collectives are the ones the NCCL group issues: one broadcast per rank slice, an int64
sum of slot words 0-10 and an fp64 sum of word 12.  The partitioned run must reproduce the
unpartitioned oracle run (permuted by pi), with the scalars equal to the exactly rounded sums.
The relabel pi below is the definition the GPU setup implements (descending out-degree, ties by
id, dangling last); tests/test_gpu_dist.py checks the GPU's pi, CSR and cuts against it.
"""
import math
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def relabel(rp, ci, deg):
    """Symmetric relabel: order = vertices by (-deg, id) with dangling last;
    rows in pi order, column ids pi(src), each row's entries in their original order."""
    n = rp.shape[0] - 1
    key = np.where(deg > 0, -deg.astype(np.int64), 1)
    order = np.lexsort((np.arange(n), key))
    pi = np.empty(n, np.int64)
    pi[order] = np.arange(n)
    lens = np.diff(rp)[order]
    rp2 = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    ci2 = np.concatenate([pi[ci[rp[v]:rp[v + 1]]] for v in order]).astype(np.int32) if ci.size else ci
    return order, pi, rp2, ci2, int((deg > 0).sum())


def _slot_allreduce(slot):
    """What the NCCL group does with an exact-accumulator slot: int64 sum of words 0-10, fp64 sum
    of word 12 (two's-complement wrap-around = the uint64 limb arithmetic)."""
    w = torch.from_numpy(slot[:11].view(np.int64).copy())
    dist.all_reduce(w)
    e = torch.from_numpy(slot[12:13].view(np.float64).copy())
    dist.all_reduce(e)
    out = slot.copy()
    out[:11] = w.numpy().view(np.uint64)
    out[12:13] = e.numpy().view(np.uint64)
    return out


def _worker(rank, world, port, scale, sweeps, out):
    import sys
    sys.path.insert(0, ROOT)
    import oracle
    from paper_2509_14211_b200 import nbg
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    src, dst = oracle.rmat_edges(scale, 8, 3)
    n = 1 << scale
    rp0, ci0, deg0 = oracle.build_csr(n, src, dst)
    order, pi, rp, ci, ncols_g = relabel(rp0, ci0, deg0)
    deg = deg0[order]                                           # out-degree of each pi position
    cuts = nbg.nbg_partition_rows(rp, world, 5 * 4)             # product rule, pi-space rows
    off, cnt = nbg.nbg_dist_exchange_plan(cuts, ncols_g)        # product exchange schedule
    lo, hi = int(cuts[rank]), int(cuts[rank + 1])
    alpha = 0.85
    dinv = np.where(deg > 0, (alpha / np.maximum(deg, 1).astype(np.float64)).astype(np.float32), np.float32(0))
    r_blk = np.full(hi - lo, np.float32(1.0 / n), np.float32)
    tele, a_n = (1 - alpha) / n, alpha / n

    def exchange(r_loc):
        y = np.zeros(ncols_g, np.float32)
        yb = (r_loc * dinv[lo:hi]).astype(np.float32)
        y[off[rank]:off[rank] + cnt[rank]] = yb[:cnt[rank]]
        t = torch.from_numpy(y)
        for q in range(world):                                  # one broadcast per slice (the NCCL group)
            if cnt[q]:
                part = t[off[q]:off[q] + cnt[q]].clone()
                dist.broadcast(part, src=q)
                t[off[q]:off[q] + cnt[q]] = part
        return t.numpy()

    ds_terms = r_blk[deg[lo:hi] == 0].astype(np.float64)
    ds = nbg.nbg_xacc_decode(_slot_allreduce(nbg.nbg_xacc_encode(ds_terms)))
    x = exchange(r_blk)
    deltas, dss = [], []
    for _ in range(sweeps):
        c = np.float32(a_n * ds + tele)
        new = oracle.sweep_rows_f32(lo, hi, rp, ci, x, c)
        d_terms = np.abs(new - r_blk).astype(np.float64)          # |r - t| in T (Fig. 6 l.290), then fp64
        ds_terms = new[deg[lo:hi] == 0].astype(np.float64)
        delta = nbg.nbg_xacc_decode(_slot_allreduce(nbg.nbg_xacc_encode(d_terms)))
        ds = nbg.nbg_xacc_decode(_slot_allreduce(nbg.nbg_xacc_encode(ds_terms)))
        deltas.append(delta)
        dss.append(ds)
        x = exchange(new)
        r_blk = new
    parts = [None] * world
    dist.all_gather_object(parts, r_blk)
    if rank == 0:
        np.save(out + ".r.npy", np.concatenate(parts))
        np.save(out + ".d.npy", np.array(deltas))
        np.save(out + ".cuts.npy", cuts)
        np.save(out + ".plan.npy", np.stack([off, cnt]))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_row_partitioned_sweeps_match_unpartitioned(tmp_path, world):
    import oracle
    scale, sweeps = 11, 15
    out = str(tmp_path / "res")
    mp.spawn(_worker, args=(world, _free_port(), scale, sweeps, out), nprocs=world, join=True)
    r = np.load(out + ".r.npy")
    deltas = np.load(out + ".d.npy")
    cuts = np.load(out + ".cuts.npy")
    off, cnt = np.load(out + ".plan.npy")
    src, dst = oracle.rmat_edges(scale, 8, 3)
    n = 1 << scale
    rp, ci, deg = oracle.build_csr(n, src, dst)
    order, pi, rp2, ci2, ncols_g = relabel(rp, ci, deg)
    ro, so, dho, _ = oracle.pagerank(rp, ci, deg, dtype=np.float32, itermax=sweeps)
    assert cuts[0] == 0 and cuts[-1] == n and 0 < cuts[1] < n
    # the slices tile [0, ncols_g) in rank order
    assert off[0] == 0 and np.array_equal(off[1:], off[:-1] + cnt[:-1]) and off[-1] + cnt[-1] == ncols_g
    # ranks (pi order): every row sum keeps its order; c differs from the oracle's only through the
    # rounding of ds (exact sum vs sequential fp64 sum), far below fp32 resolution
    assert np.max(np.abs(r - ro[order]) / ro[order]) <= 1e-6
    # delta: the exactly rounded sum of the same fp32 terms vs the oracle's sequential fp64 sum
    assert np.allclose(deltas, dho, rtol=1e-12, atol=1e-15)


def test_exchange_plan_clips_dangling_rows():
    from paper_2509_14211_b200 import nbg
    off, cnt = nbg.nbg_dist_exchange_plan(np.array([0, 5, 9, 14, 20]), 11)
    assert list(off) == [0, 5, 9, 11] and list(cnt) == [5, 4, 2, 0]
    with pytest.raises(nbg.NbgError):
        nbg.nbg_dist_exchange_plan(np.array([0, 5, 3]), 4)


def test_slot_sum_is_the_exact_sum_across_ranks():
    """Two ranks' slots summed word-wise (what the collective does) decode to the exactly rounded
    sum of the union of their terms; non-finite terms on one rank propagate (counts, not OR)."""
    from paper_2509_14211_b200 import nbg
    rng = np.random.default_rng(4)
    a = np.ldexp(rng.standard_normal(700), rng.integers(-40, 40, 700))
    b = np.ldexp(rng.standard_normal(900), rng.integers(-40, 40, 900))

    def combine(*slots):
        out = np.zeros(16, np.uint64)
        with np.errstate(over="ignore"):
            for s in slots:
                out[:11] += s[:11]
        out[12:13] = np.array([sum(s[12:13].view(np.float64)[0] for s in slots)]).view(np.uint64)
        return out

    sa, sb = nbg.nbg_xacc_encode(a), nbg.nbg_xacc_encode(b)
    assert nbg.nbg_xacc_decode(combine(sa, sb)) == math.fsum(np.concatenate([a, b]))
    assert nbg.nbg_xacc_decode(combine(sb, sa)) == nbg.nbg_xacc_decode(combine(sa, sb))
    inf = nbg.nbg_xacc_encode(np.array([1.0, np.inf]))
    assert math.isinf(nbg.nbg_xacc_decode(combine(sa, inf))) and nbg.nbg_xacc_decode(combine(sa, inf)) > 0
    ninf = nbg.nbg_xacc_encode(np.array([-np.inf]))
    assert math.isnan(nbg.nbg_xacc_decode(combine(inf, ninf)))
    assert math.isnan(nbg.nbg_xacc_decode(combine(sa, nbg.nbg_xacc_encode(np.array([np.nan])))))
