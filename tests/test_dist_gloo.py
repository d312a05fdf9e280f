"""Multi-GPU path covered on CPU (world size 2, gloo): the 1-D byte-balanced row partition
(`nbg_partition_rows`, product host code), the allgather-v assembly of the exchanged vector and
the global delta / dangling-mass reduction, with each rank's row block swept by the oracle.
The partitioned run must reproduce the unpartitioned oracle run."""
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
    rp, ci, deg = oracle.build_csr(n, src, dst)
    cuts = nbg.nbg_partition_rows(rp, world, 5 * 4)          # byte-balanced cut points
    lo, hi = int(cuts[rank]), int(cuts[rank + 1])
    alpha = 0.85
    dinv = np.where(deg > 0, (alpha / np.maximum(deg, 1).astype(np.float64)).astype(np.float32), np.float32(0))
    r_blk = np.full(hi - lo, np.float32(1.0 / n), np.float32)
    tele, a_n = (1 - alpha) / n, alpha / n
    counts = [int(cuts[q + 1] - cuts[q]) for q in range(world)]
    mx = max(counts)
    deltas = []
    for _ in range(sweeps):
        # exchange: allgather-v of y = r * dinv over the blocks (padded to the largest block)
        y_blk = (r_blk * dinv[lo:hi]).astype(np.float32)
        pad = np.zeros(mx, np.float32)
        pad[: hi - lo] = y_blk
        parts = [torch.zeros(mx, dtype=torch.float32) for _ in range(world)]
        dist.all_gather(parts, torch.from_numpy(pad))
        y = np.concatenate([parts[q].numpy()[: counts[q]] for q in range(world)])
        # dangling mass of the current ranks: local partial, global sum
        ds = torch.tensor([float(r_blk[deg[lo:hi] == 0].astype(np.float64).sum())], dtype=torch.float64)
        dist.all_reduce(ds)
        c = np.float32(a_n * float(ds.item()) + tele)
        new = oracle.sweep_rows_f32(lo, hi, rp, ci, y, c)
        d = torch.tensor([float(np.abs(new - r_blk).astype(np.float64).sum())], dtype=torch.float64)
        dist.all_reduce(d)
        deltas.append(float(d.item()))
        r_blk = new
    parts = [torch.zeros(mx, dtype=torch.float32) for _ in range(world)]
    pad = np.zeros(mx, np.float32)
    pad[: hi - lo] = r_blk
    dist.all_gather(parts, torch.from_numpy(pad))
    if rank == 0:
        r = np.concatenate([parts[q].numpy()[: counts[q]] for q in range(world)])
        np.save(out + ".r.npy", r)
        np.save(out + ".d.npy", np.array(deltas))
        np.save(out + ".cuts.npy", cuts)
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
    src, dst = oracle.rmat_edges(scale, 8, 3)
    rp, ci, deg = oracle.build_csr(1 << scale, src, dst)
    ro, so, dho, _ = oracle.pagerank(rp, ci, deg, dtype=np.float32, itermax=sweeps)
    assert cuts[0] == 0 and cuts[-1] == (1 << scale) and 0 < cuts[1] < (1 << scale)
    # per-row sums are identical; only the fp64 sum order of ds/delta differs across ranks
    assert np.max(np.abs(r - ro) / ro) <= 1e-6
    assert np.allclose(deltas, dho, rtol=1e-5, atol=1e-9)
