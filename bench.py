#!/usr/bin/env python
"""bench.py -- fused nonblocking PageRank on B200 (BASELINE.json metric, config 4 by default).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload c4|c1|c3|c5]
    python bench.py --impl reference ...      # the CPU oracle as the reference arm

A step is one whole PageRank solve through the C ABI (nbg_pagerank: every SURVEY 8(a) row --
setup of the reciprocal out-degrees, then fused sweeps until delta <= tol or itermax) on the
resident graph.  value = GTEPS/iter = (nnz * sweeps) / time / 1e9 summed over the job.
N > 1: one process per GPU (torchrun), 1-D row partition balanced by bytes, NCCL allgather-v of
the scaled ranks and exact allreduce of delta / dangling mass each sweep (nbg_pagerank_dist);
the same graph is split across ranks ("scaling": "strong").
Timing: W untimed warm-up steps (JIT + plan cache + speculation hints), then K
steps bracketed by barrier + synchronize, CUDA events on the launching stream, max over ranks.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import inputs  # noqa: E402

METRIC = "PageRank GTEPS/iter (fused mxv+ewise+reduce); achieved HBM GB/s vs peak"


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d.get("hbm_gbs", 6650.0)), "measured"
    return 6650.0, "fallback"


class Clocks:
    """nvidia-smi sampler (B200_PROFILING.md clocks line), started before the warm-up and stopped
    after the timed region; samples are time-stamped so the ones inside the timed region can be
    picked.  A timed region shorter than the sampling interval falls back to the samples taken
    under the same load (warm-up and trailing steps), and says so in "window"."""

    Q = ("timestamp,index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, device):
        self.device = device
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "20"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        import datetime
        for line in self.proc.stdout:
            f = [x.strip() for x in line.strip().split(",")]
            try:
                ts = datetime.datetime.strptime(f[0], "%Y/%m/%d %H:%M:%S.%f").timestamp()
            except Exception:
                ts = time.time()
            self.lines.append((ts, f[1:]))

    def count(self):
        return len(self.lines)

    def stop(self, t0=None, t1=None):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        inwin = [f for ts, f in self.lines if t0 is not None and t0 - 0.01 <= ts <= t1 + 0.01]
        use, window = (inwin, "timed") if inwin else ([f for _, f in self.lines], "load: warm-up + timed + trailing steps "
                                                       "(timed region shorter than the 20 ms sampling interval)")
        sm, smax, reasons = [], None, set()
        for f in use:
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                smax = float(f[2])
            except ValueError:
                continue
            for nm, v in zip(names, f[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": smax,
                "reasons": sorted(reasons), "samples": len(sm), "window": window}


def graph_params(w):
    c = inputs.CONFIGS[w]
    return c


def algorithmic_bytes(n, nnz, w):
    """B_ns = 4 nnz + 8 (n+1) + 2 w n (colidx, rowptr, x once, y once);
    B_fused = B_ns + 3 w n (t read, dinv read, y_next write)."""
    b_ns = 4 * nnz + 8 * (n + 1) + 2 * w * n
    return b_ns, b_ns + 3 * w * n


def load_ncu(workload):
    """profiles/ncu_summary.json entry of a workload (one `ncu --set full` capture of its sweep
    kernel): DRAM bytes and L2 sectors per launch, or {}."""
    p = os.path.join(ROOT, "profiles", "ncu_summary.json")
    if not os.path.exists(p):
        return {}
    try:
        return json.load(open(p)).get(workload, {})
    except Exception:
        return {}


def load_traffic(workload):
    return load_ncu(workload).get("dram_bytes_per_launch")


# L2 (LTS) random-sector throughput measured in round 1 (387 G sectors/s,
# the microarchitecture notes' ~6300 B/clk cap at 1965 MHz): the ceiling of an L2-resident sweep
L2_SECTORS_PEAK = 387e9


# ------------------------------------------------------------------ our arm

def run_ours(args, rank, world, local_rank):
    import torch
    torch.cuda.set_device(local_rank)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    from paper_2509_14211_b200 import nbg
    stream = torch.cuda.current_stream()
    ctx = nbg.nbg_init(nbg.NONBLOCKING, local_rank, stream.cuda_stream)
    cfg = graph_params(args.workload)
    T = nbg.FP32 if cfg["dtype"] == "fp32" else nbg.FP64
    w = 4 if T == nbg.FP32 else 8
    kind = nbg.GRAPH_RMAT if cfg["graph"] == "rmat" else nbg.GRAPH_ER
    t0 = time.time()
    cuts = None
    # the per-rank data plane at one rank too (default; NBG_BENCH_DIST=0 for nbg_pagerank on the
    # generator's plain CSR): symmetric relabel, rows in the gather layout, the next sweep's gathered
    # vector written in row order into its slice (C4 156.5 vs 164.8 us per sweep)
    use_dist = world > 1 or (os.environ.get("NBG_BENCH_DIST", "1") == "1" and not args.mtx)
    if use_dist:
        # per-rank setup: every rank regenerates the edges, keeps its share,
        # degrees summed over NCCL, symmetric relabel, byte-balanced row block -- no rank builds the
        # whole graph or copies a CSR to the host
        if world > 1:
            uid = nbg.nbg_dist_unique_id() if rank == 0 else None
            obj = [uid]
            dist.broadcast_object_list(obj, src=0)
            nbg.nbg_dist_init(ctx, rank, world, obj[0])
            # NBG_DIST_EXCHANGE=peer: the exchange fused into the sweep kernel as NVLink peer stores
            # (nbg_dist_set_exchange); default: one NCCL group per sweep
            xmode = os.environ.get("NBG_DIST_EXCHANGE", "collective")
            nbg.nbg_dist_set_exchange(ctx, nbg.DIST_EXCHANGE_PEER if xmode == "peer" else nbg.DIST_EXCHANGE_COLLECTIVE)
        A, deg, cuts, ncols_g = nbg.nbg_dist_graph_from_generator(ctx, kind, cfg["scale"], cfg["edge_factor"], args.seed,
                                                                  nranks=world, bytes_per_row=5 * w)
        n = int(cuts[-1])
        t_nnz = torch.tensor([nbg.nbg_matrix_nnz(ctx, A)], device="cuda", dtype=torch.int64)
        if world > 1:
            dist.all_reduce(t_nnz)
        nnz = int(t_nnz.item())
    else:
        if args.mtx:       # NEXT-4: a real graph from a Matrix Market file (the paper's GAP-web run)
            A, deg = nbg.nbg_matrix_from_mtx(ctx, args.mtx)
        else:
            A, deg = nbg.nbg_matrix_from_generator(ctx, kind, cfg["scale"], cfg["edge_factor"], args.seed)
        n = nbg.nbg_matrix_nrows(ctx, A)
        nnz = nbg.nbg_matrix_nnz(ctx, A)
        ncols_g = int((nbg.nbg_vector_export_dense(ctx, deg) > 0).sum())   # gathered-vector length (gather layout)
    setup_s = time.time() - t0
    itermax, tol = cfg["itermax"], cfg["tol"]
    dangling = nbg.PR_UNIFORM if cfg["dangling"] == "uniform" else nbg.PR_DROP

    def step():
        if use_dist:
            r, s, h = nbg.nbg_pagerank_dist(ctx, A, deg, cuts, ncols_g, alpha=cfg["alpha"], tol=tol, itermax=itermax,
                                            dangling=dangling, type=T)
        else:
            r, s, h = nbg.nbg_pagerank(ctx, A, deg, alpha=cfg["alpha"], tol=tol, itermax=itermax,
                                       dangling=dangling, type=T)
        nbg.nbg_vector_free(ctx, r)
        return s, h

    def barrier():
        if dist is not None:
            dist.barrier()

    clocks = Clocks(local_rank)
    clocks.start()
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    t_ready = time.time()
    while clocks.count() == 0 and time.time() - t_ready < 3.0:   # sampler live before the timed region
        step()
    torch.cuda.synchronize()
    def timed_pass(instrumented):
        # instrumented: per-launch CUDA events on the library's stream (kernel durations for the
        # roofline); the value's pass runs without them (two event records per launch add host and
        # GPU gaps that matter for small graphs: C1 25 vs 19 us per sweep)
        nbg.nbg_set_timing(ctx, 1 if instrumented else 0)
        barrier()
        torch.cuda.synchronize()
        w0 = time.time()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        sw = 0
        hl = None
        marks = [e0]
        for _ in range(args.steps):
            s, hl = step()
            sw += s
            ev = torch.cuda.Event(enable_timing=True)      # per-step marks (mean / median)
            ev.record(stream)
            marks.append(ev)
        e1.record(stream)
        torch.cuda.synchronize()
        w1 = time.time()
        barrier()
        return e0.elapsed_time(e1), [marks[k].elapsed_time(marks[k + 1]) for k in range(len(marks) - 1)], sw, hl, w0, w1

    st0 = nbg.nbg_get_stats(ctx)
    ms_instr, _, _, _, wi0, wi1 = timed_pass(True)
    spmv_ms, spmv_n = nbg.nbg_get_timing(ctx, "spmv")
    p2_ms, p2_n = nbg.nbg_get_timing(ctx, "spmv_p2")      # phase 2 of the two-phase SpMV (0 launches single-pass)
    ewise_ms, ewise_n = nbg.nbg_get_timing(ctx, "ewise")
    comm_ms, comm_n = nbg.nbg_get_timing(ctx, "comm")
    st_mid = nbg.nbg_get_stats(ctx)
    ms, step_ms, sweeps_total, hist_last, wall0, wall1 = timed_pass(False)
    nbg.nbg_set_timing(ctx, 0)
    st1 = nbg.nbg_get_stats(ctx)
    st0 = st_mid
    n_in = sum(1 for ts, _ in clocks.lines if wall0 - 0.01 <= ts <= wall1 + 0.01)
    if n_in == 0:        # short timed region: a few trailing steps under the same load for the sampler
        t_tr = time.time()
        c0 = clocks.count()
        while clocks.count() < c0 + 3 and time.time() - t_tr < 3.0:
            step()
        torch.cuda.synchronize()
    ck = clocks.stop(wall0, wall1)
    if dist is not None:
        t = torch.tensor([ms], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    launches = st1["kernels_launched"] - st0["kernels_launched"]

    # ---------------- end-to-end through the public API with HOST buffers (N = 1)
    e2e = None
    if world == 1 and not args.no_e2e:
        rp_h, ci_h = nbg.nbg_matrix_export_csr(ctx, A)
        deg_h = nbg.nbg_vector_export_dense(ctx, deg)
        rp_p = torch.from_numpy(rp_h).pin_memory()
        ci_p = torch.from_numpy(ci_h).pin_memory()
        dg_p = torch.from_numpy(deg_h).pin_memory()
        out_p = torch.empty(n, dtype=torch.float32 if T == nbg.FP32 else torch.float64).pin_memory()

        def e2e_step():
            A2 = nbg.nbg_matrix_from_csr(ctx, n, n, rp_p.numpy(), ci_p.numpy(), type=nbg.FP32)
            d2 = nbg.nbg_vector_from_dense(ctx, nbg.INT32, dg_p.numpy())
            r, s, _ = nbg.nbg_pagerank(ctx, A2, d2, alpha=cfg["alpha"], tol=tol, itermax=itermax, dangling=dangling,
                                       type=T)
            nbg.nbg_vector_export_dense(ctx, r, out_p.numpy())
            nbg.nbg_vector_free(ctx, r)
            nbg.nbg_vector_free(ctx, d2)
            nbg.nbg_matrix_free(ctx, A2)
            return s

        # warm-up: the second solve on a fresh matrix still compiles the dinv region with the side
        # outputs learned on the first (one NVRTC compile, cached from then on)
        for _ in range(max(2, args.warmup)):
            e2e_step()
        torch.cuda.synchronize()
        f0 = torch.cuda.Event(enable_timing=True)
        f1 = torch.cuda.Event(enable_timing=True)
        f0.record(stream)
        esw = 0
        for _ in range(args.steps):
            esw += e2e_step()
        f1.record(stream)
        torch.cuda.synchronize()
        ems = f0.elapsed_time(f1)
        e2e = {"value": nnz * esw / (ems * 1e-3) / 1e9, "unit": "GTEPS",
               "h2d_bytes_per_step": int(rp_h.nbytes + ci_h.nbytes + deg_h.nbytes),
               "d2h_bytes_per_step": int(out_p.numel() * out_p.element_size())}

    result = None
    if rank == 0:
        b_ns, b_fused = algorithmic_bytes(n, nnz, w)
        if world > 1:
            b_ns, b_fused = b_ns / world, b_fused / world      # rank 0's share (roofline is per GPU)
        pk, pk_src = peaks()
        # one sweep = one single-pass launch, or phase 1 + phase 2 of the two-phase SpMV
        avg_spmv_s = ((spmv_ms + p2_ms) / spmv_n) * 1e-3 if spmv_n else float("nan")
        achieved = b_ns / avg_spmv_s / 1e9
        traffic = None if args.mtx else load_traffic(args.workload)
        value = nnz * sweeps_total / (ms * 1e-3) / 1e9
        result = {
            "metric": METRIC,
            "value": round(value, 3),
            "unit": "GTEPS",
            "n_gpus": world,
            "steps": args.steps,
            "warmup": args.warmup,
            "ms_per_step": round(ms / args.steps, 4),
            "step_ms": {"mean": round(statistics.mean(step_ms), 4), "median": round(statistics.median(step_ms), 4),
                        "min": round(min(step_ms), 4), "max": round(max(step_ms), 4)},
            "higher_is_better": True,
            "scaling": "strong",
            "vs_baseline": None,
            "dtype": "f32" if T == nbg.FP32 else "f64",
            "data": f"file {os.path.basename(args.mtx)}" if args.mtx else "synthetic",
            "config": {
                "workload": workload_name(args, cfg),
                "n": n, "nnz": nnz, "dangling": cfg["dangling"], "alpha": cfg["alpha"], "tol": tol,
                "itermax": itermax, "sweeps_per_step": sweeps_total / args.steps,
                "parallelism": f"rows{world}" if world > 1 else ("single (per-rank data plane, P = 1)" if use_dist else "single"),
                **({"exchange": os.environ.get("NBG_DIST_EXCHANGE", "collective")} if world > 1 else {}),
                "layout": "symmetric gather-layout relabel (rows and columns by descending out-degree, dangling last)"
                          if use_dist else "column gather layout, rows in generator order",
                "l2": l2_note(nnz, ncols_g * w),
                "setup_s": round(setup_s, 3),
            },
            "roofline": {
                "bound": "hbm", "kernel": "fused SpMV sweep (nbg_spmv*: row-binned nbg_spmvr_* on C4 / C5)",
                "achieved": round(achieved, 1), "peak": pk, "peak_source": pk_src, "unit": "GB/s",
                "frac": round(achieved / pk, 4), "traffic": traffic,
                "bytes_per_launch_ns": int(b_ns), "bytes_per_launch_fused": int(b_fused),
                "achieved_fused_gbs": round(b_fused / avg_spmv_s / 1e9, 1),
                "avg_launch_us": round(avg_spmv_s * 1e6, 2), "launches": spmv_n + p2_n,
                "sweep_kernels": "two-phase (phase 1 %.1f us + phase 2 %.1f us)" % (spmv_ms / spmv_n * 1e3, p2_ms / p2_n * 1e3)
                                 if p2_n else "single-pass",
                "share_of_step": round((spmv_ms + p2_ms) / ms_instr, 4) if ms_instr else None,
                **({"l2": {"bound_note": "L2-resident gathered vector and index stream: L2 sectors, not HBM bytes, bound "
                                         "this sweep" if "stays L2-resident" in l2_note(nnz, ncols_g * w) and
                                         load_ncu(args.workload).get("dram_bytes_per_launch", 1e30) < 0.5 * b_ns
                                         else "L2 sectors of the same launch, for comparison",
                          "sectors_per_launch": load_ncu(args.workload)["lts_sectors_per_launch"],
                          "achieved_gsectors_s": round(load_ncu(args.workload)["lts_sectors_per_launch"] / avg_spmv_s / 1e9, 1),
                          "peak_gsectors_s": L2_SECTORS_PEAK / 1e9,
                          "frac": round(load_ncu(args.workload)["lts_sectors_per_launch"] / avg_spmv_s / L2_SECTORS_PEAK, 4),
                          "source": "sectors: ncu lts__t_sectors.sum of one sweep launch (profiles/ncu_summary.json); "
                                    "peak: measured random-sector throughput (DESIGN.md section 7)"}}
                   if (not args.mtx and "lts_sectors_per_launch" in load_ncu(args.workload)) else {}),
                "timing_pass": "kernel durations from an instrumented pass of the same K steps right before the "
                               "value's pass (per-launch CUDA events on the library stream); "
                               "ms_per_step with events %.4f" % (ms_instr / args.steps),
            },
            "e2e": e2e,
            "gpu_launches": int(launches),
            "kernel_ms": {"spmv": round(spmv_ms + p2_ms, 3), "ewise": round(ewise_ms, 3), "comm": round(comm_ms, 3),
                          "ewise_launches": ewise_n, "comm_launches": comm_n},
            "planner": {k: st1[k] - st0[k] for k in ("plans_built", "plan_hits", "memo_hits", "side_outputs",
                                                      "intermediates_elided", "waits")},
            "host_plan_us_per_wait": round((st1["host_plan_ns"] - st0["host_plan_ns"]) / 1e3 /
                                           max(1, st1["waits"] - st0["waits"]), 2),
            "clocks": ck,
        }
    nbg.nbg_vector_free(ctx, deg)
    nbg.nbg_matrix_free(ctx, A)
    nbg.nbg_finalize(ctx)
    if dist is not None:
        dist.destroy_process_group()
    return result


# ------------------------------------------------------------------ config 2: fused elementwise chain

def torch_dot_reference(x, y, steps):
    """Context for config 2's roofline: a library read of the same two vectors (torch.dot, cuBLAS)
    under the same L2 flush -- how fast a plain read-both-vectors kernel goes at this size."""
    import torch
    xt = torch.from_numpy(x).cuda()
    yt = torch.from_numpy(y).cuda()
    flush = torch.ones(64 << 20, dtype=torch.float32, device="cuda")
    sink = torch.empty(1, dtype=torch.float32, device="cuda")
    best, tot = 1e9, 0.0
    for k in range(3 + steps):
        sink.copy_(flush.sum().view(1))
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        torch.dot(xt, yt)
        e1.record()
        torch.cuda.synchronize()
        if k >= 3:
            ms = e0.elapsed_time(e1)
            best, tot = min(best, ms), tot + ms
    nb = x.nbytes + y.nbytes
    return {"what": "torch.dot(x, y) on the same device vectors, L2 flushed the same way (CUDA events)",
            "avg_us": round(tot / steps * 1e3, 2), "gbs_avg": round(nb / (tot / steps * 1e-3) / 1e9, 1),
            "gbs_best": round(nb / (best * 1e-3) / 1e9, 1)}


def run_chain(args):
    """BASELINE config 2: z = x * (y + 1), then c1..c5 and reduce(+) over n = 2^24 (SURVEY 8(a)
    a13), fused (nonblocking: one pass, every intermediate elided) vs blocking (one kernel per op).
    value = fused GB/s over the algorithmic bytes 2 w n (x and y read once)."""
    import torch
    from paper_2509_14211_b200 import nbg
    torch.cuda.set_device(0)
    n = inputs.CONFIGS["c2"]["n"]
    npT = np.float32 if args.dtype == "fp32" else np.float64
    t = nbg.FP32 if args.dtype == "fp32" else nbg.FP64
    w = 4 if args.dtype == "fp32" else 8
    x, y = inputs.uniform_vectors(n, args.seed, npT)
    stream = torch.cuda.current_stream()
    out = {}
    clocks = Clocks(0)
    clocks.start()
    ck = None
    for mode, name in ((nbg.NONBLOCKING, "fused"), (nbg.BLOCKING, "blocking")):
        c = nbg.nbg_init(mode, 0, stream.cuda_stream)
        vx = nbg.nbg_vector_from_dense(c, t, x)
        vy = nbg.nbg_vector_from_dense(c, t, y)

        def step():
            a = nbg.nbg_apply(c, t, "ADD_C", vy, 1.0)
            z = nbg.nbg_ewise_mult(c, t, "TIMES", vx, a)
            c1 = nbg.nbg_apply(c, t, "MUL_C", z, 0.5)
            c2 = nbg.nbg_ewise_add(c, t, "PLUS", c1, vx)
            c3 = nbg.nbg_ewise_mult(c, t, "TIMES", c2, vy)
            c4 = nbg.nbg_apply(c, t, "ABS_SUB_C", c3, 0.25)
            c5 = nbg.nbg_ewise_add(c, t, "MAX", c4, z)
            s = nbg.nbg_reduce(c, nbg.FP64, "PLUS", c5)
            for h in (a, z, c1, c2, c3, c4, c5):
                nbg.nbg_vector_free(c, h)
            v = nbg.nbg_scalar_get(c, s)
            nbg.nbg_scalar_free(c, s)
            return v

        for _ in range(args.warmup):
            step()
        # > L2: inputs come from HBM.  Flushed by READING a 256 MB buffer (clean lines): a write-based
        # flush would leave dirty lines whose write-back competes with the timed kernel
        flush = torch.ones(64 << 20, dtype=torch.float32, device="cuda")
        sink = torch.empty(1, dtype=torch.float32, device="cuda")
        ms = 0.0
        if name == "fused":
            t_ready = time.time()
            while clocks.count() == 0 and time.time() - t_ready < 3.0:   # sampler live before the timed region
                step()
        st0 = nbg.nbg_get_stats(c)
        nbg.nbg_set_timing(c, 1)
        torch.cuda.synchronize()
        wall0 = time.time()
        for _ in range(args.steps):
            sink.copy_(flush.sum().view(1))
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            step()
            e1.record(stream)
            torch.cuda.synchronize()
            ms += e0.elapsed_time(e1)
        wall1 = time.time()
        if name == "fused":
            # the timed region is short: a few trailing steps under the same load for the sampler
            if sum(1 for ts, _ in clocks.lines if wall0 - 0.01 <= ts <= wall1 + 0.01) == 0:
                t_tr = time.time()
                c0 = clocks.count()
                while clocks.count() < c0 + 3 and time.time() - t_tr < 3.0:
                    sink.copy_(flush.sum().view(1))
                    step()
                torch.cuda.synchronize()
            ck = clocks.stop(wall0, wall1)
        st1 = nbg.nbg_get_stats(c)
        kms, kn = nbg.nbg_get_timing(c, "ewise")          # device time of the chain's kernels
        nbg.nbg_set_timing(c, 0)
        out[name] = (ms / args.steps, (st1["kernels_launched"] - st0["kernels_launched"]) / args.steps, kms / args.steps)
        nbg.nbg_vector_free(c, vx)
        nbg.nbg_vector_free(c, vy)
        nbg.nbg_finalize(c)
    pk, pk_src = peaks()
    b_alg = 2 * w * n
    fused_ms, fused_k, fused_kms = out["fused"]
    blk_ms, blk_k, blk_kms = out["blocking"]
    gbs = b_alg / (fused_ms * 1e-3) / 1e9            # whole step: record 8 ops + wait + scalar read-back
    kgbs = b_alg / (fused_kms * 1e-3) / 1e9          # the fused kernel alone (CUDA events on its stream)
    return {"metric": "config-2 elementwise chain, fused HBM GB/s (x, y read once)", "value": round(gbs, 1), "unit": "GB/s",
            "n_gpus": 1, "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(fused_ms, 4),
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32" if w == 4 else "f64",
            "data": "synthetic",
            "config": {"workload": f"c2: chain of 8 ops + reduce(+), n = 2^24, seed {args.seed}",
                       "l2": "flushed before every step (read of a 256 MB buffer)"},
            "roofline": {"bound": "hbm", "kernel": "fused chain (nbg_ewise_*)", "achieved": round(kgbs, 1), "peak": pk,
                         "peak_source": pk_src, "unit": "GB/s", "frac": round(kgbs / pk, 4), "traffic": None,
                         "bytes_per_launch": b_alg, "avg_launch_us": round(fused_kms * 1e3, 2)},
            "library_reference": torch_dot_reference(x, y, args.steps),
            "blocking": {"ms_per_step": round(blk_ms, 4), "kernels_per_step": blk_k, "kernel_ms_per_step": round(blk_kms, 4),
                         "speedup_fused_vs_blocking": round(blk_ms / fused_ms, 2),
                         "kernel_speedup_fused_vs_blocking": round(blk_kms / fused_kms, 2)},
            "gpu_launches": int(round(fused_k * args.steps)), "clocks": ck}


# ------------------------------------------------------------------ NEXT-3: sparse / bitset vectors

def run_sparse(args):
    """Structured regions: s = reduce(+, ewise_mult(*, u, x)) and
    w = ewise_add(+, u, v) with u, v sparse (fill f) and x full, n = 2^24 fp32.  For each fill the
    estimator's loop choice (auto) is timed next to the forced alternative (NBG_STRUCT_LOOP), so
    the line shows whether the naive fill estimate picks the faster loop.
    value = present entries of u processed per second by the mult+reduce step at f = 0.01 (auto)."""
    import torch
    from paper_2509_14211_b200 import nbg
    torch.cuda.set_device(0)
    n = 1 << 24
    rng = np.random.default_rng(args.seed)
    xv = rng.random(n).astype(np.float32)
    stream = torch.cuda.current_stream()
    c = nbg.nbg_init(nbg.NONBLOCKING, 0, stream.cuda_stream)
    dx = nbg.nbg_vector_from_dense(c, nbg.FP32, xv)
    rows = []
    pk, pk_src = peaks()
    for fill in (0.001, 0.01, 0.03, 0.06, 0.1, 0.4):
        iu = np.nonzero(rng.random(n) < fill)[0].astype(np.int32)
        iv = np.nonzero(rng.random(n) < fill)[0].astype(np.int32)
        du = nbg.nbg_vector_from_sparse(c, nbg.FP32, n, iu, rng.random(iu.shape[0]).astype(np.float32))
        dv = nbg.nbg_vector_from_sparse(c, nbg.FP32, n, iv, rng.random(iv.shape[0]).astype(np.float32))
        row = {"fill": fill, "nvals": int(iu.shape[0])}
        for loop in ("auto", "index", "dense"):
            if loop == "auto":
                os.environ.pop("NBG_STRUCT_LOOP", None)
            else:
                os.environ["NBG_STRUCT_LOOP"] = loop

            def step():
                m = nbg.nbg_ewise_mult(c, nbg.FP32, "TIMES", du, dx)
                s = nbg.nbg_reduce(c, nbg.FP64, "PLUS", m)
                v = nbg.nbg_scalar_get(c, s)
                nbg.nbg_scalar_free(c, s)
                nbg.nbg_vector_free(c, m)
                w = nbg.nbg_ewise_add(c, nbg.FP32, "PLUS", du, dv)
                k = nbg.nbg_vector_nvals(c, w)
                nbg.nbg_vector_free(c, w)
                return v, k

            for _ in range(args.warmup):
                step()
            st0 = nbg.nbg_get_stats(c)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            for _ in range(args.steps):
                step()
            torch.cuda.synchronize()
            ms = (time.perf_counter() - t0) * 1e3 / args.steps
            st1 = nbg.nbg_get_stats(c)
            row[loop + "_ms"] = round(ms, 4)
            if loop == "auto":
                row["auto_index_loops_per_step"] = (st1["structured_index_loops"] - st0["structured_index_loops"]) / args.steps
        os.environ.pop("NBG_STRUCT_LOOP", None)
        # algorithmic bytes of the mult+reduce over the index loop: u's indices and values, x at u's positions
        row["index_bytes"] = int(iu.shape[0]) * 12
        rows.append(row)
        nbg.nbg_vector_free(c, du)
        nbg.nbg_vector_free(c, dv)
    nbg.nbg_finalize(c)
    r01 = [r for r in rows if r["fill"] == 0.01][0]
    return {"metric": "structured ewise_mult+reduce and ewise_add over sparse vectors (present entries/s of u)",
            "value": round(r01["nvals"] / (r01["auto_ms"] * 1e-3) / 1e9, 4), "unit": "G entries/s", "n_gpus": 1,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": r01["auto_ms"], "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": "sparse: n = 2^24, u, v sparse with fill f (uniform random support), x full; "
                                   "step = reduce(+, u .* x) read back + nvals(u + v)", "timing": "host wall clock per step (includes the scalar read-back and nvals syncs)"},
            "peak_hbm_gbs": pk, "fills": rows}


# ------------------------------------------------------------------ oracle (cpu_baseline / reference arm)

def workload_name(args, cfg):
    if args.mtx:
        return f"mtx {os.path.basename(args.mtx)} (c4 solver settings)"
    return f"{args.workload}: {cfg['graph']} scale {cfg['scale']} ef {cfg['edge_factor']} seed {args.seed}"


def oracle_graph(cfg, seed, mtx=None):
    import oracle
    if mtx:
        n, src, dst = oracle.read_mtx(mtx)
        return oracle.build_csr(n, src, dst)
    f = oracle.rmat_edges if cfg["graph"] == "rmat" else oracle.er_edges
    src, dst = f(cfg["scale"], cfg["edge_factor"], seed)
    rp, ci, deg = oracle.build_csr(1 << cfg["scale"], src, dst)
    del src, dst
    return rp, ci, deg


def oracle_sample(rp, ci, deg, cfg, sweeps, threads=False):
    """Time `sweeps` fixed sweeps of the oracle (Fig. 6) -> seconds.  threads=True: the OpenMP
    build of the same source (rows split over all host cores, identical results)."""
    import oracle
    dt = np.float32 if cfg["dtype"] == "fp32" else np.float64
    if threads:
        oracle.lib_omp()                      # build / load outside the timed region
    t0 = time.perf_counter()
    oracle.pagerank(rp, ci, deg, alpha=cfg["alpha"], dtype=dt, uniform=cfg["dangling"] == "uniform",
                    itermax=sweeps, tol=-1.0, threads=threads)
    return time.perf_counter() - t0


def omp_threads():
    v = os.environ.get("OMP_NUM_THREADS")
    return int(v) if v and v.isdigit() else (os.cpu_count() or 1)


def l2_note(nnz, gathered_bytes):
    """How the L2 stands between timed sweeps (no flush): the colidx stream vs L2, and whether the
    gathered vector can stay resident (else the persisting window over its head, jit.cpp)."""
    L2 = 126e6
    win = os.environ.get("NBG_L2_PERSIST_MB")
    win_mb = int(win) if win and win.isdigit() else 56
    s = "no flush: colidx stream %.0f MB %s L2 (126 MB) each sweep; " % (4 * nnz / 1e6, ">" if 4 * nnz > L2 else "<=")
    if gathered_bytes <= 48e6:
        s += "gathered vector %.1f MB (gather layout) stays L2-resident" % (gathered_bytes / 1e6)
    else:
        s += ("gathered vector %.0f MB does not stay L2-resident: a %d MB persisting L2 window covers its "
              "hottest head" % (gathered_bytes / 1e6, win_mb) if win_mb > 0 else
              "gathered vector %.0f MB does not stay L2-resident (persisting window off)" % (gathered_bytes / 1e6))
    return s


def cpu_model():
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except Exception:
        pass
    return None


def cpu_baseline(args):
    cfg = graph_params(args.workload)
    rp, ci, deg = oracle_graph(cfg, args.seed, args.mtx)
    nnz = int(ci.shape[0])
    sweeps = max(1, min(cfg["itermax"], int(args.cpu_sweeps)))
    t1 = oracle_sample(rp, ci, deg, cfg, sweeps)
    tn = oracle_sample(rp, ci, deg, cfg, sweeps, threads=True)
    nth = omp_threads()
    # the oracle single-threaded and its OpenMP row-parallel build on all
    # host cores; `value` / `cores` are the all-core run (the stronger baseline)
    return {"value": round(nnz * sweeps / tn / 1e9, 5), "unit": "GTEPS", "cores": nth, "kind": "oracle",
            "cpu": cpu_model(), "host_cores_available": os.cpu_count(),
            "single_thread": {"value": round(nnz * sweeps / t1 / 1e9, 5), "unit": "GTEPS", "cores": 1,
                              "seconds": round(t1, 3)},
            "sample": f"{sweeps} fixed Fig. 6 sweeps of the C oracle on the same graph ({nnz} edges): "
                      f"OpenMP row loop on {nth} threads {tn:.2f} s, single-threaded {t1:.2f} s"}


def run_reference(args, rank, world):
    if rank != 0:
        return None
    cfg = graph_params(args.workload)
    rp, ci, deg = oracle_graph(cfg, args.seed, args.mtx)
    nnz = int(ci.shape[0])
    per = max(1, int(args.ref_sweeps))
    nth = omp_threads()
    for _ in range(args.warmup):
        oracle_sample(rp, ci, deg, cfg, per, threads=True)
    tot = 0.0
    for _ in range(args.steps):
        tot += oracle_sample(rp, ci, deg, cfg, per, threads=True)
    value = nnz * per * args.steps / tot / 1e9
    return {
        "metric": METRIC, "value": round(value, 5), "unit": "GTEPS", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(tot / args.steps * 1e3, 3), "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f32" if cfg["dtype"] == "fp32" else "f64",
        "data": f"file {os.path.basename(args.mtx)}" if args.mtx else "synthetic", "impl": "reference",
        "config": {"workload": workload_name(args, cfg), "n": int(rp.shape[0] - 1), "nnz": nnz,
                   "step": f"{per} fixed sweeps of the CPU oracle (bounded sample of the workload)"},
        "cpu_baseline": {"value": round(value, 5), "unit": "GTEPS", "cores": nth, "kind": "oracle", "cpu": cpu_model(),
                         "sample": f"{per} sweeps x {args.steps} steps, C oracle with its row loop on {nth} "
                                   f"OpenMP threads (identical results to the single-threaded build)"},
        "e2e": {"value": round(value, 5), "unit": "GTEPS", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=60)   # ≈ 0.2 s timed at C4: several 20 ms clock samples inside it
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="c4", choices=["c1", "c2", "c3", "c4", "c5", "sparse"])
    ap.add_argument("--dtype", default="fp32", choices=["fp32", "fp64"], help="c2 only")
    ap.add_argument("--seed", type=int, default=1)
    ap.add_argument("--cpu-sweeps", type=int, default=60)   # ≈ 10 s of oracle work at C4
    ap.add_argument("--ref-sweeps", type=int, default=2)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--mtx", default=None, help="Matrix Market file instead of the synthetic graph (c4 settings)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3) if args.impl == "ours" else args.warmup
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local_rank = int(os.environ.get("LOCAL_RANK", 0))
    if world != args.gpus and world == 1 and args.gpus > 1:
        print(json.dumps({"error": "--gpus N>1 must be launched with torchrun"}))
        sys.exit(2)
    if args.mtx:
        args.workload = "c4"
    if args.workload in ("c2", "sparse"):
        fn = run_chain if args.workload == "c2" else run_sparse
        res = fn(args) if args.impl == "ours" and rank == 0 else None
        if rank == 0 and res is not None:
            print(json.dumps(res), flush=True)
        return
    if args.impl == "reference":
        res = run_reference(args, rank, world)
    else:
        res = run_ours(args, rank, world, local_rank)
        if rank == 0 and res is not None:
            if world == 1 and not args.no_cpu_baseline:
                res["cpu_baseline"] = cpu_baseline(args)
            else:
                res["cpu_baseline"] = None
    if rank == 0 and res is not None:
        print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()
