#!/usr/bin/env python
"""Headline benchmark: approximate n x n products/sec at n=8192 (BASELINE.json config C4).

C4 = mixed decompositions, fp32: A approximated by rSVD rank 64 (sigma_i=(i+1)^-1.5, Haar U,V),
B by its top 64 cycles (N(0,1e-3^2) residue + 64 dominant N(0,1) cycles), first-order product.
One "step" = one full approximate product (decomposition of both operands + multiply) on inputs
already resident in HBM. Inputs (2 x 256 MiB fp32) are larger than the 126 MB L2, so no flush is
needed between steps.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
  torchrun --nproc-per-node N bench.py --gpus N ...      (one independent product per GPU)

Multi-GPU: every rank runs its own products (replicas, weak scaling); value = products of all
ranks / max-over-ranks device time. The row-sharded single-product path is not used here.
`--impl reference` times the reference's CPU algorithm (the numpy oracle port in oracle/, the
only bench leg allowed to execute it) on this host's cores, rank 0 only.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "approx n×n products/sec at n=8192 (rel err vs exact AB); % of HBM/FP64-TC roofline"
N_DEFAULT, K_SVD, K_CYC = 8192, 64, 64
# Stage markers recorded by the C4 plan (capi.cu run_mixed_f32_umma): 0 start | hi stream: 1 B
# decomposed, 2 gather done | lo stream: 3 Y, 4 QR, 5 Bm, 9 W GEMM, 6 W | main: 7 M += Q.W, 8 end.
N_MARKS = 10
SPANS = {  # name -> (start marker, end marker); "join" = the later of markers 2 and 7
    "B: cycle norms+select+extract [hi]": (0, 1),
    "M = A.Bhat (persistent row gather) [hi]": (1, 2),
    "Y = A.Omega (tcgen05 TF32) [lo]": (0, 3),
    "QR (CholeskyQR) [lo]": (3, 4),
    "Bm = Q^T A (+||Bm||^2) [lo]": (4, 5),
    "W0 = Bm.B (tcgen05 TF32) [lo]": (5, 9),
    "W = W0 - Bm.Bhat (TF32-exact gather) [lo]": (9, 6),
    "M += Q.W (+||M||^2; each tile waits for its gather rows) [lo]": (6, 7),
    "after the join (fixed-order sums)": ("join", 8),
}
GATHER_SPAN = "M = A.Bhat (persistent row gather) [hi]"


def gather_capture():
    """DRAM traffic and L1 data-pipe load of the dominant kernel from the newest committed
    `ncu --set full` capture (profiles/r*_gather_ncu.txt), or None."""
    import glob
    import re
    files = sorted(glob.glob(os.path.join(ROOT, "profiles", "r[0-9][0-9]_gather_ncu.txt")))
    if not files:
        return None
    vals = {}
    for line in open(files[-1]):
        m = re.match(r"(\S+)\s+([0-9.]+)\s*(\S*)", line)
        if m:
            scale = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0}.get(m.group(3), 1.0)
            vals[m.group(1)] = float(m.group(2)) * scale
    try:
        traffic = vals["dram__bytes_read.sum"] + vals["dram__bytes_write.sum"]
        pipe = vals["l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed"] / 100.0
        grid = vals["launch__grid_size"]
    except KeyError:
        return None
    return {"file": os.path.relpath(files[-1], ROOT), "traffic": traffic,
            "l1_datapath_frac_active_sms": pipe * 148.0 / min(148.0, grid)}


def hbm_peak():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


# ------------------------------------------------------------------------------------------
# clocks during the timed region (NVML, 10 ms sampling)
# ------------------------------------------------------------------------------------------
class ClockSampler:
    REASONS = {"hw_slowdown": 0x8, "hw_thermal_slowdown": 0x40, "sw_thermal_slowdown": 0x20,
               "sw_power_cap": 0x4, "hw_power_brake_slowdown": 0x80}

    def __init__(self, index):
        self.samples, self.reasons, self.ok = [], set(), False
        self._stop = threading.Event()
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception:
            self.max = None

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                r = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for name, bit in self.REASONS.items():
                    if r & bit:
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(0.01)

    def __enter__(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        if self.ok:
            self._stop.set()
            self.t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max, "reasons": sorted(self.reasons),
                    "samples": 0}
        return {"sm_mhz": float(statistics.median(self.samples)), "sm_max_mhz": self.max,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


# ------------------------------------------------------------------------------------------
# multi-rank plumbing (replicas: every rank runs its own products; no data-path collective)
# ------------------------------------------------------------------------------------------
def replica_seed(rank: int) -> int:
    """Operand seed of rank `rank`'s replica: independent inputs per GPU."""
    return 1234 + 17 * rank


def max_over_ranks(x: float, world: int, device) -> float:
    """Max of a per-rank scalar over the job: the slowest rank sets the job's time."""
    import torch
    import torch.distributed as dist
    t = torch.tensor([float(x)], device=device, dtype=torch.float64)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def job_throughput(units_per_rank: int, world: int, seconds_max: float) -> float:
    """Whole-job rate: the units all ranks processed over the max-over-ranks time."""
    return world * units_per_rank / seconds_max


# ------------------------------------------------------------------------------------------
# synthetic C4 operands, generated on the device (torch Philox, seeded per rank)
# ------------------------------------------------------------------------------------------
def gen_c4(n, seed, dev):
    import torch
    g = torch.Generator(device=dev).manual_seed(seed)
    sig = (torch.arange(n, device=dev, dtype=torch.float64) + 1.0) ** -1.5

    def haar():
        Q, R = torch.linalg.qr(torch.randn(n, n, generator=g, device=dev, dtype=torch.float64))
        d = torch.sign(torch.diagonal(R))
        d[d == 0] = 1.0
        return Q * d

    Q1 = haar()
    Q2 = haar()
    A = ((Q1 * sig) @ Q2.T).float().contiguous()
    del Q1, Q2
    B = 1e-3 * torch.randn(n, n, generator=g, device=dev, dtype=torch.float32)
    J = torch.randperm(n, generator=g, device=dev)[:K_CYC]
    i = torch.arange(n, device=dev)
    for j in J.tolist():
        B[i, (i - j) % n] += torch.randn(n, generator=g, device=dev, dtype=torch.float32)
    torch.cuda.synchronize()
    return A, B


# ------------------------------------------------------------------------------------------
# CPU reference (oracle port) on a bounded sample: full decomposition + a block of output rows
# ------------------------------------------------------------------------------------------
def cpu_reference_sample(A64, B64, seed, rows_per_step, steps, warmup):
    import oracle as O
    n = A64.shape[0]
    t0 = time.perf_counter()
    Mr, rep = O.mixed_first_order_multiply(A64, B64, K_SVD, K_CYC, 1, seed,
                                           rows=np.arange(rows_per_step))
    first = time.perf_counter() - t0
    t_dec = rep["t_decompose"]
    t_rows = []
    rng = np.random.default_rng(seed)
    for s in range(warmup + steps):
        r0 = int(rng.integers(0, n - rows_per_step))
        rows = np.arange(r0, r0 + rows_per_step)
        U_t = time.perf_counter()
        _cpu_rows(A64, B64, rep, seed, rows)
        if s >= warmup:
            t_rows.append(time.perf_counter() - U_t)
    per_row = statistics.median(t_rows) / rows_per_step
    # first call = decomposition + V^T B + the first row block; remaining rows at the sampled rate
    t_prod = first + per_row * (n - rows_per_step)
    return {"t_decompose_s": t_dec, "t_rows_median_s": statistics.median(t_rows),
            "rows_per_step": rows_per_step, "t_product_est_s": t_prod, "first_call_s": first,
            "M_rows0": Mr, "selected_b": rep["selected_b"]}


_CACHE = {}


def _cpu_rows(A, B, rep, seed, rows):
    """Output rows of the oracle's mixed product given its (cached) decomposition."""
    import oracle as O
    from oracle import apx_oracle as OX
    key = id(A)
    if key not in _CACHE:
        U, s, V, fa = O.rsvd(A, K_SVD, np.random.default_rng([seed, 0]), 0)
        Jb, lb, _, _, _ = O.cycle_decompose(B, K_CYC)
        _CACHE[key] = (U, s, V, Jb, lb, V.T @ B)
    U, s, V, Jb, lb, VtB = _CACHE[key]
    Us = U[rows] * s
    dA = A[rows] - Us @ V.T
    return Us @ VtB + OX._cycle_right_apply(dA, Jb, lb)


def run_reference(args, rank):
    if rank != 0:
        return
    import torch
    n = args.n
    # same synthetic distributions, host-generated at reduced cost (Haar via numpy QR is slow at
    # n=8192, so the reference arm uses the device generator when a GPU is present)
    if torch.cuda.is_available():
        A, B = gen_c4(n, 1234, torch.device("cuda", 0))
        A64, B64 = A.double().cpu().numpy(), B.double().cpu().numpy()
        del A, B
    else:
        import oracle as O
        A64 = O.gen_haar_spectrum(n, (np.arange(n) + 1.0) ** -1.5, 1).astype(np.float32).astype(np.float64)
        B64 = O.gen_cycle_operand(n, K_CYC, 2).astype(np.float32).astype(np.float64)
    r = cpu_reference_sample(A64, B64, 7, args.cpu_rows, args.steps, args.warmup)
    v = 1.0 / r["t_product_est_s"]
    cores = os.cpu_count()
    sample = (f"full decomposition of both operands ({r['t_decompose_s']:.2f} s, first call "
              f"{r['first_call_s']:.2f} s) + "
              f"{args.cpu_rows} output rows per step ({r['t_rows_median_s']:.3f} s median over "
              f"{args.steps} steps), extrapolated linearly to {n} rows")
    line = {"metric": METRIC, "value": v, "unit": "products/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * r["t_product_est_s"],
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "impl": "reference",
            "config": {"workload": "C4 mixed rSVD(k=64) x cycles(k=64) first-order product, n=8192",
                       "n": n, "k_svd": K_SVD, "k_cyc": K_CYC, "order": 1},
            "cpu_baseline": {"value": v, "unit": "products/s", "cores": cores, "kind": "port",
                             "sample": sample},
            "e2e": {"value": v, "unit": "products/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------------------------------
# our arm
# ------------------------------------------------------------------------------------------
def run_ours(args, rank, world, local_rank):
    import torch
    import torch.distributed as dist
    import paper_2504_19308_b200 as P
    from paper_2504_19308_b200 import _native as N

    dev = torch.device("cuda", local_rank)
    torch.cuda.set_device(dev)
    n = args.n
    A, B = gen_c4(n, replica_seed(rank), dev)
    seed = 7
    omega = torch.from_numpy(P.cycle.draw_sketch(n, K_SVD, seed)).to(dev, torch.float32)
    M = torch.empty(n, n, device=dev, dtype=torch.float32)
    split3 = bool(args.split3)

    def step(out=M):
        return P.mixed_product_device(A, B, K_SVD, K_CYC, 1, omega, 0, None, split3, out=out)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()

    # ---- timed region: K products on resident inputs; only the gather's two stage events
    # (markers 1, 2, recorded on the gather's stream) are live here ----
    import ctypes
    lib = N.lib()
    gev = [[torch.cuda.Event(enable_timing=True) for _ in range(2)] for _ in range(args.steps)]
    for row in gev:
        for e in row:
            e.record()
    torch.cuda.synchronize()
    gptr = [(ctypes.c_void_p * N_MARKS)(*([None, row[0].cuda_event, row[1].cuda_event] + [None] * (N_MARKS - 3)))
            for row in gev]
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    l0 = lib.apx_launch_count()
    with ClockSampler(local_rank) as clk:
        start.record()
        for s in range(args.steps):
            lib.apx_set_stage_events(gptr[s], N_MARKS)
            step()
        lib.apx_set_stage_events(None, 0)
        end.record()
        torch.cuda.synchronize()
    launches = lib.apx_launch_count() - l0
    gather_ms_timed = statistics.mean(row[0].elapsed_time(row[1]) for row in gev)

    # ---- full stage breakdown: the same K products again, all stage events (outside the timing) ----
    nst = N_MARKS
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(nst)] for _ in range(args.steps)]
    for row in evs:  # torch creates the underlying cudaEvent_t lazily, on first record
        for e in row:
            e.record()
    torch.cuda.synchronize()
    ev_ptrs = [(ctypes.c_void_p * nst)(*[e.cuda_event for e in row]) for row in evs]
    for s in range(args.steps):
        lib.apx_set_stage_events(ev_ptrs[s], nst)
        step()
    lib.apx_set_stage_events(None, 0)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ms_max = max_over_ranks(start.elapsed_time(end), world, dev)
    def span_ms(row, a, b):
        t = [0.0] + [row[0].elapsed_time(row[i]) for i in range(1, nst)]
        ta = max(t[2], t[7]) if a == "join" else t[a]
        return t[b] - ta

    stage_ms = {name: statistics.mean(span_ms(evs[s], a, b) for s in range(args.steps))
                for name, (a, b) in SPANS.items()}

    # ---- e2e: public API with pinned host buffers (H2D inputs, D2H result, every step) ----
    # MixedPipeline (the host-to-host serving API): each product copies its full A, B in and its
    # full M out; product i's D2H overlaps product i+1's H2D (PCIe is full duplex) and its compute.
    e2e = None
    if not args.no_e2e:
        Ah = torch.empty((n, n), dtype=torch.float32, pin_memory=True)
        Bh = torch.empty((n, n), dtype=torch.float32, pin_memory=True)
        Mh = [torch.empty((n, n), dtype=torch.float32, pin_memory=True) for _ in range(3)]
        Ah.copy_(A)
        Bh.copy_(B)
        pipe = P.MixedPipeline(n, K_SVD, K_CYC, 1, depth=3, split3=split3)
        for i in range(2):
            pipe.result(pipe.submit(Ah, Bh, seed, out=Mh[i % 3]))
        e2e_steps = max(4, min(args.steps, 24))
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        tickets = [pipe.submit(Ah, Bh, seed, out=Mh[i % 3]) for i in range(e2e_steps)]
        reps = [pipe.result(t)[1] for t in tickets]
        torch.cuda.synchronize()
        te = max_over_ranks(time.perf_counter() - t0, world, dev)
        assert all(r.selected_b == reps[0].selected_b for r in reps)
        e2e = {"value": job_throughput(e2e_steps, world, te), "unit": "products/s",
               "h2d_bytes_per_step": 2 * n * n * 4 + n * K_SVD * 4,
               "d2h_bytes_per_step": n * n * 4 + N.NSCALARS * 8 + K_CYC * 4,
               "steps": e2e_steps, "ms_per_step": 1e3 * te / e2e_steps,
               "path": "paper_2504_19308_b200.MixedPipeline.submit/result (pinned host tensors, depth 3)"}
        del pipe

    # ---- correctness side-channel (outside every timed region) ----
    r = step()
    torch.cuda.synchronize()
    sel_gpu = r["sel_b"].tolist()
    exact = (A.double() @ B.double())
    rel_exact = float(torch.linalg.norm(M.double() - exact) / torch.linalg.norm(exact))
    del exact
    s = r["scalars"].tolist()

    line = None
    if rank == 0:
        peak, peak_kind = hbm_peak()
        gather_ms = gather_ms_timed  # mean gather span inside the timed region
        cap = gather_capture()
        alg_bytes = 8.0 * n * n  # A read + M write (fp32); Q.W accumulates onto it afterwards
        achieved = alg_bytes / (gather_ms * 1e-3) / 1e9
        total_alg_bytes = 24.0 * n * n  # SURVEY §8(d) C4 algorithmic bytes per product
        line = {
            "metric": METRIC, "value": job_throughput(args.steps, world, ms_max * 1e-3), "unit": "products/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": ms_max / args.steps, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": "C4 mixed rSVD(k=64) x cycles(k=64) first-order product, n=8192",
                       "n": n, "k_svd": K_SVD, "k_cyc": K_CYC, "order": 1, "power_iterations": 0,
                       "gemm": "3xTF32 mma.sync" if split3 else "tcgen05 kind::tf32 (TMA, warp-specialized)",
                       "parallelism": f"replicas x{world} (one product per GPU per step)",
                       "l2": "inputs larger than L2 (2 x 256 MiB fp32); no flush"},
            "clocks": clk.summary(), "e2e": e2e, "gpu_launches": int(launches),
            "roofline": {"bound": "hbm", "kernel": "cycle_right_gather (M = A.Bhat, persistent)",
                         "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak,
                         "traffic": cap["traffic"] if cap else None, "peak_kind": peak_kind,
                         "alg_bytes_per_launch": alg_bytes,
                         "datapath": ({"l1_wavefront_frac_active_sms": cap["l1_datapath_frac_active_sms"],
                                       "source": cap["file"]} if cap else None),
                         "note": ("the gather is bound by the SM load datapath (k*n^2 fp32 operands at "
                                  "128 B/clk/SM), not HBM: see datapath and DESIGN.md section 4")},
            "whole_product_hbm_frac": (total_alg_bytes / (ms_max / args.steps * 1e-3) / 1e9) / peak,
            "stages_ms": stage_ms,
            "rel_err_vs_exact": rel_exact,
            "norms": {"norm_da": math.sqrt(max(0, s[0] - s[2])), "norm_db": math.sqrt(max(0, s[1] - s[3]))},
        }
    # ---- CPU baseline (rank 0, N=1 only): oracle port on a bounded sample ----
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        A64 = A.double().cpu().numpy()
        B64 = B.double().cpu().numpy()
        cb = cpu_reference_sample(A64, B64, seed, args.cpu_rows, 3, 1)
        line["cpu_baseline"] = {
            "value": 1.0 / cb["t_product_est_s"], "unit": "products/s", "cores": os.cpu_count(),
            "kind": "port",
            "sample": (f"oracle port: full decomposition ({cb['t_decompose_s']:.2f} s) + "
                       f"{args.cpu_rows}-row output blocks ({cb['t_rows_median_s']:.3f} s median), "
                       f"extrapolated to {n} rows; numpy BLAS on all cores, rolls single-threaded")}
        rows = np.arange(args.cpu_rows)
        Mg = M[: args.cpu_rows].double().cpu().numpy()
        line["parity_vs_oracle_rows"] = {
            "rows": int(args.cpu_rows),
            "rel": float(np.linalg.norm(Mg - cb["M_rows0"]) / np.linalg.norm(cb["M_rows0"])),
            "selection_equal": sel_gpu == list(cb["selected_b"]), "tol": 1e-4}
    if rank == 0:
        print(json.dumps(line), flush=True)


def run_sharded(args, rank, world, local_rank):
    """--shard rows: ONE C4 product per step for the whole job, its rows of A and M split over the
    ranks (sharded.mixed_product_rows; NCCL all-reduces of the Gram matrices, Q^T A and two norms).
    Strong scaling: value = products/s of the job (max-over-ranks time)."""
    import torch
    import torch.distributed as dist
    import paper_2504_19308_b200 as P
    from paper_2504_19308_b200 import _native as N
    from paper_2504_19308_b200 import sharded as S

    dev = torch.device("cuda", local_rank)
    torch.cuda.set_device(dev)
    n = args.n
    A, B = gen_c4(n, 1234, dev)  # the same operands on every rank; each keeps its rows of A
    r0, r1 = S.row_range(n, world, rank)
    A_rows = A[r0:r1].contiguous()
    omega = torch.from_numpy(P.cycle.draw_sketch(n, K_SVD, 7)).to(dev, torch.float32)
    M_rows = torch.empty(r1 - r0, n, device=dev, dtype=torch.float32)

    def reduce(t):
        if world > 1:
            dist.all_reduce(t)

    def step():
        return S._drive(S.mixed_rows_steps(A_rows, B, K_SVD, K_CYC, 1, omega, out=M_rows), reduce)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    l0 = N.lib().apx_launch_count()
    with ClockSampler(local_rank) as clk:
        start.record()
        for _ in range(args.steps):
            r = step()
        end.record()
        torch.cuda.synchronize()
    launches = N.lib().apx_launch_count() - l0
    S.check_breakdown(r)
    if world > 1:
        dist.barrier()
    ms_max = max_over_ranks(start.elapsed_time(end), world, dev)
    # correctness side-channel: these rows against the exact product's rows, selections equal
    exact = A_rows.double() @ B.double()
    err2 = torch.tensor([float(torch.linalg.norm(M_rows.double() - exact) ** 2),
                         float(torch.linalg.norm(exact) ** 2)], device=dev, dtype=torch.float64)
    del exact
    sel = r["sel_b"].to(torch.int64)
    if world > 1:
        dist.all_reduce(err2)
        sels = [torch.empty_like(sel) for _ in range(world)]
        dist.all_gather(sels, sel)
        same = all(torch.equal(x, sels[0]) for x in sels)
    else:
        same = True
    if rank == 0:
        s = r["scalars"].tolist()
        line = {
            "metric": METRIC, "value": args.steps / (ms_max * 1e-3), "unit": "products/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": ms_max / args.steps, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": "C4 mixed rSVD(k=64) x cycles(k=64) first-order product, n=8192",
                       "n": n, "k_svd": K_SVD, "k_cyc": K_CYC, "order": 1, "power_iterations": 0,
                       "parallelism": f"rows x{world} (one product per step, row blocks of A and M per rank)",
                       "l2": "inputs larger than L2 (256 MiB B per rank); no flush"},
            "clocks": clk.summary(), "gpu_launches": int(launches),
            "rel_err_vs_exact": math.sqrt(err2[0].item() / err2[1].item()),
            "selection_equal_across_ranks": same,
            "norms": {"norm_da": math.sqrt(max(0, s[0] - s[2])), "norm_db": math.sqrt(max(0, s[1] - s[3]))},
        }
        print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--n", type=int, default=N_DEFAULT)
    ap.add_argument("--cpu-rows", type=int, default=128)
    ap.add_argument("--split3", type=int, default=0)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--shard", default="replicas", choices=["replicas", "rows"],
                    help="replicas: one product per GPU (weak scaling, default); rows: one product per "
                         "step split by rows over the GPUs (strong scaling)")
    args = ap.parse_args()
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local_rank = int(os.environ.get("LOCAL_RANK", 0))
    if args.impl == "reference":
        run_reference(args, rank)
        return
    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local_rank)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    try:
        if args.shard == "rows":
            run_sharded(args, rank, world, local_rank)
        else:
            run_ours(args, rank, world, local_rank)
    finally:
        if world > 1:
            import torch.distributed as dist
            dist.destroy_process_group()


if __name__ == "__main__":
    main()
