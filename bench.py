#!/usr/bin/env python
"""Benchmarks: approximate n x n products/sec (BASELINE.json metric) on the BASELINE configs.

Headline (default, ``--config c4``): C4 = mixed decompositions, fp32, n = 8192: A approximated by
rSVD rank 64 (sigma_i=(i+1)^-1.5, Haar U,V), B by its top 64 cycles (N(0,1e-3^2) residue + 64
dominant N(0,1) cycles), first-order product. One "step" = one full approximate product
(decomposition of both operands + multiply) on inputs already resident in HBM. Inputs (2 x 256
MiB fp32) are larger than the 126 MB L2, so no flush is needed between steps.

  python bench.py [--config c4|c1|c2|c3|c5|c5c] [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
  torchrun --nproc-per-node N bench.py --gpus N ...

Multi-GPU (one process per GPU, NCCL):
  * c4 (default for N > 1): ONE product per step, sharded by row blocks of A and M over the ranks
    (BASELINE config 4; sharded.mixed_product_rows: all-gathers of the small factors with a fixed
    rank-order sum) -- strong scaling. ``--shard replicas``: one independent product per GPU.
  * c5: row-sharded cycle product at N < 8 (strong), one product per GPU at N = 8 (BASELINE
    config 5: "one product per GPU at 8 GPUs and row-block sharding at 1/2/4").
  * c1, c2, c3, c5c: independent products per GPU (replicas, weak scaling).
``--impl reference`` times the reference's CPU algorithm (the numpy oracle port in oracle/, the
only bench leg allowed to execute it) on this host's cores, rank 0 only, one full product per
step (C5: a row sample -- its full product does not fit host memory).
"""

from __future__ import annotations

import argparse
import glob
import json
import math
import os
import re
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "approx n×n products/sec at n=8192 (rel err vs exact AB); % of HBM/FP64-TC roofline"
N_DEFAULT, K_SVD, K_CYC = 8192, 64, 64
WORKLOADS = {
    "c4": "C4 mixed rSVD(k=64) x cycles(k=64) first-order product, n=8192",
    "c1": "C1 rSVD-truncated product fp64 n=512 (k=32, p=8, q=2, order 0)",
    "c2": "C2 cycle-truncated product fp64 n=2048 (k=32, order 1)",
    "c3": "C3 circulant product fp64 n=4096 (k=16, order 1)",
    "c5": "C5 cycle product fp32 n=32768 (k=128, order 1; 128 cycles + 32 circulant terms + noise)",
    "c5c": "C5 secondary: circulant product (k=32, order 1) on the C5 operands, fp64 on the device",
}
# Stage markers recorded by the C4 plan (capi.cu run_mixed_f32_umma): 0 start | hi stream: 1 B
# decomposed, 2 gather done | lo stream: 3 Y, 4 QR, 5 Bm, 9 W GEMM, 6 W | main: 7 M += Q.W, 8 end.
N_MARKS = 18
# C4 stage markers (capi.cu run_mixed_f32_resid / run_mixed_f32_umma): name -> (start, end);
# "join" = the later of markers 2 and 7. GATHER_MARKS: the gather's own span (timed region).
SPANS = {
    "B: cycle norms+select+extract+f16 lambda' [hi]": (0, 1),
    "Y = A.Omega (tcgen05 TF32) [lo]": (0, 3),
    "QR (CholeskyQR) [lo]": (3, 4),
    "Bm = Q^T A (+||A||^2, ||Bm||^2; A tiles rounded to TF32) [lo]": (4, 5),
    "dA = A - [Q|Q].[Bm_hi;Bm_lo] -> scaled f16 (tcgen05, fused epilogue) [lo]": (5, 10),
    "M = dA.Bhat (persistent f16 row gather) [hi]": (11, 2),
    "W0 = Bm.B (tcgen05 TF32) [lo]": (10, 9),
    "W = W0 - Bm.Bhat_tf32 + Bm.Bhat (gathers), hi/lo split [lo]": (9, 6),
    "M += [Q|Q].[W_hi;W_lo] (+||M||^2; each tile waits for its gather rows) [lo]": (6, 7),
    "after the join (fixed-order sums)": ("join", 8),
}
SPANS_DIRECT = {
    "B: cycle norms+select+extract [hi]": (0, 1),
    "M = A.Bhat (persistent row gather) [hi]": (1, 2),
    "Y = A.Omega (tcgen05 TF32) [lo]": (0, 3),
    "QR (CholeskyQR) [lo]": (3, 4),
    "Bm = Q^T A (+||Bm||^2; operands rounded to TF32) [lo]": (4, 5),
    "W0 = Bm.B (tcgen05 TF32) [lo]": (10, 9),
    "W = W0 - Bm.Bhat (TF32-exact gather) [lo]": (9, 6),
    "M += Q.W (+||M||^2; each tile waits for its gather rows) [lo]": (6, 7),
    "after the join (fixed-order sums)": ("join", 8),
}


# ------------------------------------------------------------------------------------------
# peaks, captures, host description
# ------------------------------------------------------------------------------------------
def hbm_peak():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"]), "measured (MEASURED_PEAKS.json)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


def pipe_peaks():
    """Pipe peaks measured on this pool by tools/peaks.cu (newest profiles/r*_pipe_peaks.jsonl)."""
    files = sorted(glob.glob(os.path.join(ROOT, "profiles", "r[0-9][0-9]_pipe_peaks.jsonl")))
    best = {}
    for f in files[-1:]:
        for line in open(f):
            try:
                d = json.loads(line)
            except ValueError:
                continue
            for k, v in d.items():
                if isinstance(v, (int, float)):
                    best[k] = max(best.get(k, 0.0), float(v))
        best["source"] = os.path.relpath(f, ROOT)
    return best


def gather_capture():
    """DRAM traffic and L1 data-pipe load of the dominant kernel from the newest committed
    `ncu --set full` capture (profiles/r*_gather_ncu.txt), or None."""
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


# committed `ncu --set full` summaries of each config's dominant kernels (tools/ncu_summary.py format)
NCU_FILES = {
    "c1": ["profiles/r02c_cqr2_c1_ncu.txt"],
    "c2": ["profiles/r02e_c2_cycle_right_gather_ncu.txt", "profiles/r02e_c2_cycle_left_gather_ncu.txt"],
    "c3": ["profiles/r02e_c3_circ_left2_r16_ncu.txt", "profiles/r02e_c3_circ_right2_r16_ncu.txt",
           "profiles/r02e_c3_circ_decompose_r16_ncu.txt"],
    "c5": ["profiles/r01_seg_gather_ncu.txt"],
    "c5c": ["profiles/r02c_fft4_pass1_r16_ncu.txt", "profiles/r02c_fft4_pass2_r16_ncu.txt"],
}


def ncu_limiters(cfg):
    """Per dominant kernel of `cfg`: which unit the committed ncu capture shows it bound by (L1
    data pipe, DRAM, FP64 / FMA pipe utilisation as fractions of their peaks). Static evidence
    read from profiles/, not a measurement of this run."""
    out = []
    for rel_path in NCU_FILES.get(cfg, []):
        path = os.path.join(ROOT, rel_path)
        if not os.path.exists(path):
            continue
        vals, name = {}, None
        for line in open(path):
            if line.startswith("Kernel Name"):
                name = line[len("Kernel Name"):].strip().split("(")[0].replace("void ", "")
            m = re.match(r"(\S+)\s+([0-9.]+)\s*(\S*)", line)
            if m:
                vals[m.group(1)] = float(m.group(2))
        pct = lambda k: (vals[k] / 100.0) if k in vals else None  # noqa: E731
        out.append({"kernel": name,
                    "l1_data_pipe_frac": pct("l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed"),
                    "dram_frac": pct("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"),
                    "fp64_pipe_frac": pct("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"),
                    "fma_pipe_frac": pct("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active"),
                    "source": rel_path})
    return out or None


def host_info():
    """CPU model, core count and BLAS threading of the host the CPU leg runs on."""
    model = None
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for line in out.splitlines():
            if line.startswith("Model name"):
                model = line.split(":", 1)[1].strip()
    except Exception:
        pass
    blas = None
    try:
        from threadpoolctl import threadpool_info
        blas = [{"api": d.get("internal_api"), "threads": d.get("num_threads")} for d in threadpool_info()]
    except Exception:
        pass
    return {"cpu_model": model, "cores": os.cpu_count(), "blas": blas,
            "OPENBLAS_NUM_THREADS": os.environ.get("OPENBLAS_NUM_THREADS"),
            "note": "np.fft / fancy indexing single-threaded; BLAS and the oracle's row blocks (a thread pool) use all cores"}


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
            return {"sm_mhz": None, "sm_max_mhz": self.max, "reasons": sorted(self.reasons), "samples": 0}
        return {"sm_mhz": float(statistics.median(self.samples)), "sm_max_mhz": self.max,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


# ------------------------------------------------------------------------------------------
# multi-rank plumbing
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


def gen_c4(n, seed, dev):
    """C4 operands on the device (paper_2504_19308_b200.genmat.c4_operands)."""
    from paper_2504_19308_b200 import genmat
    return genmat.c4_operands(n, seed, dev, K_CYC)


def _timed_region(step, steps, world, dev, local_rank, lib):
    """W warm-up already done by the caller; K steps bracketed by barrier + synchronize, timed
    with CUDA events on the current stream. Returns (ms of this rank, launches, clocks)."""
    import torch
    import torch.distributed as dist
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    l0 = lib.apx_launch_count()
    with ClockSampler(local_rank) as clk:
        start.record()
        for _ in range(steps):
            step()
        end.record()
        torch.cuda.synchronize()
    return start.elapsed_time(end), lib.apx_launch_count() - l0, clk.summary()


# ------------------------------------------------------------------------------------------
# CPU legs (oracle port: the reference's algorithm in numpy; cpu_baseline and --impl reference)
# ------------------------------------------------------------------------------------------
def cpu_c4_product(A64, B64, seed):
    """One full C4 product by the oracle port (rSVD + cycle decomposition + all n output rows)."""
    import oracle as O
    t0 = time.perf_counter()
    M, rep = O.mixed_first_order_multiply(A64, B64, K_SVD, K_CYC, 1, seed)
    return time.perf_counter() - t0, M, rep


def cpu_product(cfg, ops):
    """One full product of config `cfg` by the oracle port on host operands; returns (s, M, rep)."""
    import oracle as O
    t0 = time.perf_counter()
    if cfg == "c1":
        A, B, t = ops
        M, rep = O.svd_first_order_multiply(A, B, None, 0, t, power_iterations=2, components=32, oversampling=8)
    elif cfg == "c2":
        A, B = ops
        M, rep = O.cycle_first_order_multiply(A, B, 32, 1)
    elif cfg == "c3":
        A, B = ops[:2]
        # near-tie protocol: the operands' conjugate-pair spectra tie exactly at
        # the selection boundary, so the oracle runs with the GPU's selections when they are given
        sel = ops[2] if len(ops) > 2 else (None, None)
        M, rep = O.circulant_first_order_multiply(A, B, 16, 1, sel[0], sel[1])
    else:
        raise ValueError(cfg)
    return time.perf_counter() - t0, M, rep


# ------------------------------------------------------------------------------------------
# C4 (headline): one product per step on this GPU
# ------------------------------------------------------------------------------------------
def run_c4(args, rank, world, local_rank):
    import ctypes

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

    direct = args.plan == "direct"
    spans = SPANS_DIRECT if direct else SPANS
    g0 = 1 if direct else 11  # marker opening the gather's span

    def step(out=M):
        return P.mixed_product_device(A, B, K_SVD, K_CYC, 1, omega, 0, None, False, out=out, direct=direct)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()

    # ---- timed region: K products on resident inputs; only the gather's two stage events
    # (markers 1, 2, recorded on the gather's stream) are live here ----
    lib = N.lib()
    gev = [[torch.cuda.Event(enable_timing=True) for _ in range(2)] for _ in range(args.steps)]
    for row in gev:
        for e in row:
            e.record()
    torch.cuda.synchronize()
    def gather_marks(row):
        m = [None] * N_MARKS
        m[g0], m[2] = row[0].cuda_event, row[1].cuda_event
        return (ctypes.c_void_p * N_MARKS)(*m)

    gptr = [gather_marks(row) for row in gev]
    it = iter(range(args.steps))

    def timed_step():
        s = next(it)
        lib.apx_set_stage_events(gptr[s], N_MARKS)
        step()

    ms, launches, clocks = _timed_region(timed_step, args.steps, world, dev, local_rank, lib)
    lib.apx_set_stage_events(None, 0)
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
    ms_max = max_over_ranks(ms, world, dev)

    def span_ms(row, a, b):
        t = [0.0] + [row[0].elapsed_time(row[i]) for i in range(1, nst)]
        ta = max(t[2], t[7]) if a == "join" else t[a]
        return t[b] - ta

    stage_ms = {name: statistics.mean(span_ms(evs[s], a, b) for s in range(args.steps))
                for name, (a, b) in spans.items()}
    # critical-path timeline of the residual plan (hi stream), ms from the product's start
    timeline = None
    if not direct:
        marks = {"Y start": 17, "Y": 3, "QR gram": 12, "QR cholinv": 13, "QR apply": 14, "QR pass 2 (gated)": 15, "QR done": 4,
                 "Bm GEMM": 16, "Bm finalize": 5, "dA": 10, "gather start": 11, "gather end": 2, "end": 8}
        timeline = {k: round(statistics.mean(evs[s][0].elapsed_time(evs[s][i]) for s in range(args.steps)), 4)
                    for k, i in marks.items()}

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
        pipe = P.MixedPipeline(n, K_SVD, K_CYC, 1, depth=3)
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
               "path": "paper_2504_19308_b200.MixedPipeline.submit/result (pinned host tensors, depth 3; "
                       "the sketch Omega is drawn on the host per product, inside this timing)"}
        del pipe, Ah, Bh, Mh

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
        pk = pipe_peaks()
        cap = gather_capture()
        # gather: (direct) fp32 A read + M write, Q.W accumulated onto M afterwards; (residual plan)
        # f16 dA read + M write, Q.W accumulated afterwards
        alg_bytes = (8.0 if direct else 6.0) * n * n
        achieved = alg_bytes / (gather_ms_timed * 1e-3) / 1e9
        total_alg_bytes = 24.0 * n * n  # SURVEY §8(d) C4 algorithmic bytes per product
        # one shared-memory operand per FMA (k n^2 FMAs): fp32 (direct) or f16 (residual plan)
        lds_bytes = (4.0 if direct else 2.0) * K_CYC * n * n
        lds_achieved = lds_bytes / (gather_ms_timed * 1e-3) / 1e12
        lds_peak = pk.get("lds64_tbs" if direct else "lds128_tbs")
        from paper_2504_19308_b200.cycle import _norms
        nA, nB, ndA, ndB, nM = _norms(s, n * n)
        line = {
            "metric": METRIC, "value": job_throughput(args.steps, world, ms_max * 1e-3), "unit": "products/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": ms_max / args.steps, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": WORKLOADS["c4"], "n": n, "k_svd": K_SVD, "k_cyc": K_CYC, "order": 1,
                       "power_iterations": 0, "gemm": "tcgen05 kind::tf32 (TMA, warp-specialized)",
                       "plan": ("direct: M = A.Bhat (fp32 gather) + Q.W" if direct else
                                "residual: M = Q.(Bm.B) + dA.Bhat, dA and lambda' in scaled f16 (FHFMA, fp32 "
                                "accumulation), Q.(.) as a K=2l TF32 hi/lo GEMM"),
                       "parallelism": f"replicas x{world} (one product per GPU per step)",
                       "l2": "inputs larger than L2 (2 x 256 MiB fp32); no flush",
                       "sketch": "Omega drawn once on the host (numpy default_rng([7,0]), the reference's "
                                 "stream) outside the device-timed region; e2e draws it per product"},
            "clocks": clocks, "e2e": e2e, "gpu_launches": int(launches),
            "roofline": {"bound": "hbm",
                         "kernel": ("cycle_right_gather (M = A.Bhat, persistent)" if direct else
                                    "cycle_gather_f16_kernel (M = dA.Bhat, persistent, f16 operands)"),
                         "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                         "traffic": cap["traffic"] if cap else None, "peak_kind": peak_kind,
                         "alg_bytes_per_launch": alg_bytes,
                         "datapath": {"resource": "shared-memory load bandwidth (the gather's real limiter)",
                                      "alg_bytes_per_launch": lds_bytes, "achieved_tbs": lds_achieved,
                                      "peak_tbs": lds_peak, "frac": (lds_achieved / lds_peak) if lds_peak else None,
                                      "peak_source": pk.get("source"),
                                      "l1_wavefront_frac_active_sms": cap["l1_datapath_frac_active_sms"] if cap else None,
                                      "ncu_source": cap["file"] if cap else None},
                         "note": ("the gather is bound by the SM load datapath (k*n^2 fp32 operands at "
                                  "128 B/clk/SM), not HBM: see datapath and DESIGN.md section 4")},
            "whole_product_hbm_frac": (total_alg_bytes / (ms_max / args.steps * 1e-3) / 1e9) / peak,
            "stages_ms": stage_ms,
            "timeline_ms": timeline,
            "rel_err_vs_exact": rel_exact,
            "norms": {"norm_a": nA, "norm_b": nB, "norm_da": ndA, "norm_db": ndB, "norm_m": nM},
        }
    # ---- CPU baseline (rank 0, N=1 only): one full product by the oracle port, timed ----
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        A64 = A.double().cpu().numpy()
        B64 = B.double().cpu().numpy()
        t_cpu, Mo, ro = cpu_c4_product(A64, B64, seed)
        hi = host_info()
        line["cpu_baseline"] = {
            "value": 1.0 / t_cpu, "unit": "products/s", "cores": hi["cores"], "kind": "port",
            "sample": (f"one full n={n} product by the oracle port (all {n} rows; decomposition "
                       f"{ro['t_decompose']:.2f} s), timed with perf_counter"),
            "host": hi}
        Mg = M.double().cpu().numpy()
        row_err = np.linalg.norm(Mg - Mo, axis=1) / np.linalg.norm(Mo, axis=1)
        line["parity_vs_oracle"] = {
            "rows": n, "rel": float(np.linalg.norm(Mg - Mo) / np.linalg.norm(Mo)),
            "worst_row_rel": float(row_err.max()), "selection_equal": sel_gpu == list(ro["selected_b"]),
            "tol": 1e-4, "norm_da_oracle": ro["norm_da"], "norm_db_oracle": ro["norm_db"]}
        del A64, B64, Mo, Mg
    if rank == 0:
        print(json.dumps(line), flush=True)


# ------------------------------------------------------------------------------------------
# C4 sharded by rows (BASELINE config 4 at N > 1): one product per step for the whole job
# ------------------------------------------------------------------------------------------
def run_c4_rows(args, rank, world, local_rank):
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
    del A
    omega = torch.from_numpy(P.cycle.draw_sketch(n, K_SVD, 7)).to(dev, torch.float32)
    M_rows = torch.empty(r1 - r0, n, device=dev, dtype=torch.float32)
    group = dist.group.WORLD if world > 1 else None

    def reduce(t):
        if world > 1:
            S.ordered_sum(t, group)

    res = {}

    def step():
        res["r"] = S._drive(S.mixed_rows_steps(A_rows, B, K_SVD, K_CYC, 1, omega, out=M_rows), reduce)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    ms, launches, clocks = _timed_region(step, args.steps, world, dev, local_rank, N.lib())
    r = res["r"]
    S.check_breakdown(r)
    if world > 1:
        dist.barrier()
    ms_max = max_over_ranks(ms, world, dev)

    # ---- e2e: every step copies this rank's rows of A and the whole B in from pinned host memory
    # and its rows of M back out ----
    e2e = None
    if not args.no_e2e:
        Ah = torch.empty(A_rows.shape, dtype=torch.float32, pin_memory=True)
        Bh = torch.empty(B.shape, dtype=torch.float32, pin_memory=True)
        Mh = torch.empty(M_rows.shape, dtype=torch.float32, pin_memory=True)
        Ah.copy_(A_rows)
        Bh.copy_(B)
        Ad, Bd = torch.empty_like(A_rows), torch.empty_like(B)

        def e2e_step():
            Ad.copy_(Ah, non_blocking=True)
            Bd.copy_(Bh, non_blocking=True)
            S._drive(S.mixed_rows_steps(Ad, Bd, K_SVD, K_CYC, 1, omega, out=M_rows), reduce)
            Mh.copy_(M_rows, non_blocking=True)

        e2e_step()
        torch.cuda.synchronize()
        e2e_steps = max(4, min(args.steps, 12))
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        for _ in range(e2e_steps):
            e2e_step()
        torch.cuda.synchronize()
        te = max_over_ranks(time.perf_counter() - t0, world, dev)
        e2e = {"value": e2e_steps / te, "unit": "products/s",
               "h2d_bytes_per_step": (r1 - r0) * n * 4 + n * n * 4,
               "d2h_bytes_per_step": (r1 - r0) * n * 4,
               "bytes_note": "per rank; B is replicated, so every rank copies all of it",
               "steps": e2e_steps, "ms_per_step": 1e3 * te / e2e_steps,
               "path": "sharded.mixed_rows_steps on H2D-copied operands, D2H of the rank's rows"}
        del Ah, Bh, Mh, Ad, Bd
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
        from paper_2504_19308_b200.cycle import _norms
        nA, nB, ndA, ndB, nM = _norms(s, n * n)
        line = {
            "metric": METRIC, "value": args.steps / (ms_max * 1e-3), "unit": "products/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": ms_max / args.steps, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": WORKLOADS["c4"], "n": n, "k_svd": K_SVD, "k_cyc": K_CYC, "order": 1,
                       "power_iterations": 0,
                       "parallelism": f"rows x{world} (one product per step, row blocks of A and M per rank)",
                       "exchanges": "all-gather + fixed rank-order sum of two 64x64 Gram matrices, Q^T A "
                                    "(64 x n fp32) and two norms (sharded.ordered_sum)",
                       "l2": "inputs larger than L2 (256 MiB B per rank); no flush"},
            "clocks": clocks, "e2e": e2e, "gpu_launches": int(launches),
            "rel_err_vs_exact": math.sqrt(err2[0].item() / err2[1].item()),
            "selection_equal_across_ranks": same,
            "norms": {"norm_a": nA, "norm_b": nB, "norm_da": ndA, "norm_db": ndB, "norm_m": nM},
        }
        print(json.dumps(line), flush=True)


# ------------------------------------------------------------------------------------------
# secondary configs (parity cases; measured with the same contract)
# ------------------------------------------------------------------------------------------
def _secondary_setup(cfg, rank, world, dev):
    """Device operands and the step of config `cfg`: returns dict(step, units, roofline inputs,
    public-API e2e call, host operands for the CPU leg)."""
    import torch

    import paper_2504_19308_b200 as P
    from paper_2504_19308_b200 import _native as N
    from paper_2504_19308_b200 import circulant as PC
    from paper_2504_19308_b200 import genmat as G

    seed = replica_seed(rank)
    out = {}
    if cfg == "c1":
        n, nb = 512, 128
        sig = 0.9 ** np.arange(n)
        A = torch.stack([G.haar_spectrum(n, sig, [seed, 2 * t], dev) for t in range(nb)])
        B = torch.stack([G.haar_spectrum(n, sig, [seed, 2 * t + 1], dev) for t in range(nb)])
        oa = torch.from_numpy(np.stack([np.random.default_rng([t, 0]).standard_normal((n, 40)) for t in range(nb)]))
        ob = torch.from_numpy(np.stack([np.random.default_rng([t, 1]).standard_normal((n, 40)) for t in range(nb)]))
        bt = P.SvdProductBatch(A, B, 40, 32, 40, 32, 2, 0, oa, ob, streams=32)
        out.update(step=bt.run, units=nb, n=n, dtype="f64", bound="fp64-tensor (DMMA)",
                   flops=nb * (24.0 * n * n * 40 + 2.0 * n * n * 32), peak_key="fp64_dmma_mma_sync_tflops",
                   note=f"{nb} independent products per step (SvdProductBatch: one CUDA graph, 32 streams)",
                   host_ops=lambda: (A[0].cpu().numpy(), B[0].cpu().numpy(), 0),
                   api=lambda Ah, Bh: P.svd_first_order_multiply(Ah, Bh, None, 0, 0, power_iterations=2,
                                                                 components=32, oversampling=8),
                   dev_out=lambda: bt.M[0], keep=(A, B, bt))
    elif cfg == "c2":
        n, nb = 2048, 16
        ops = [(G.cycle_operand(n, 32, seed * 100 + 2 * t, dev)[0], G.cycle_operand(n, 32, seed * 100 + 2 * t + 1, dev)[0])
               for t in range(nb)]
        Ms = [torch.empty(n, n, dtype=torch.float64, device=dev) for _ in range(nb)]
        calls = [(lambda a, b, m: (lambda: P.cycle_product_device(a, b, 32, 32, 1, out=m)))(a, b, m)
                 for (a, b), m in zip(ops, Ms)]
        bt = P.GraphBatch(calls, streams=8)
        out.update(step=bt.replay, units=nb, n=n, dtype="f64", bound="hbm", bytes=nb * 40.0 * n * n,
                   note=f"{nb} independent products per step (GraphBatch: one CUDA graph, 8 streams)",
                   host_ops=lambda: (ops[0][0].cpu().numpy(), ops[0][1].cpu().numpy()),
                   api=lambda Ah, Bh: P.cycle_first_order_multiply(Ah, Bh, 32, 1),
                   dev_out=lambda: Ms[0], keep=(ops, Ms, bt))
    elif cfg == "c3":
        n = 4096
        A = G.circulant_operand(n, 16, seed * 2, dev)
        B = G.circulant_operand(n, 16, seed * 2 + 1, dev)
        M = torch.empty(n, n, dtype=torch.complex128, device=dev)
        res = {}

        def step():
            res["r"] = PC.circulant_product_device(A, B, N.APX_F64, 16, 1, out=M)

        out.update(step=step, units=1, n=n, dtype="f64", bound="fp64 (DFMA)", flops=12.5e9,
                   peak_key="fp64_dfma_tflops", bytes_alt=80.0 * n * n,
                   note="one product per step; roofline T* = max(80n^2 B / HBM, 12.5 GFLOP / DFMA) (SURVEY §8(d))",
                   host_ops=lambda: (A.cpu().numpy(), B.cpu().numpy(),
                                     (res["r"]["sel_a"].tolist(), res["r"]["sel_b"].tolist()) if "r" in res
                                     else (None, None)),
                   api=lambda Ah, Bh: P.circulant_first_order_multiply(Ah, Bh, 16, 1),
                   dev_out=lambda: M, keep=(A, B, M, res))
    elif cfg in ("c5", "c5c"):
        n = 32768
        A, _ = G.c5_operand(n, 128, 32, seed, 0, dev)
        B, _ = G.c5_operand(n, 128, 32, seed, 1, dev)
        if cfg == "c5":
            M = torch.empty(n, n, dtype=torch.float32, device=dev)
            out.update(step=lambda: P.cycle_product_device(A, B, 128, 128, 1, out=M), units=1, n=n, dtype="f32",
                       bound="fp32 (FFMA) / shared-memory datapath", flops=4.0 * 128 * n * n,
                       peak_key="fp32_ffma2_tflops", lds_bytes=2 * 4.0 * 128 * n * n,
                       note="one product per step (the full oracle does not fit host memory)",
                       host_ops=None, api=None, dev_out=lambda: M, keep=(A, B, M))
        else:
            A64, B64 = A.double(), B.double()
            del A, B
            torch.cuda.empty_cache()
            M = torch.empty(n, n, dtype=torch.complex128, device=dev)
            out.update(step=lambda: PC.circulant_product_device(A64, B64, N.APX_F64, 32, 1, out=M), units=1, n=n,
                       dtype="f64", bound="hbm", bytes=40.0 * n * n,
                       note="one product per step (SURVEY §8(d): ~40 n^2 B); four-step transforms through "
                            "global memory",
                       host_ops=None, api=None, dev_out=lambda: M, keep=(A64, B64, M))
    return out


def run_secondary(args, rank, world, local_rank):
    import torch
    import torch.distributed as dist

    from paper_2504_19308_b200 import _native as N

    cfg = args.config
    dev = torch.device("cuda", local_rank)
    torch.cuda.set_device(dev)
    st = _secondary_setup(cfg, rank, world, dev)
    for _ in range(args.warmup):
        st["step"]()
    torch.cuda.synchronize()
    ms, launches, clocks = _timed_region(st["step"], args.steps, world, dev, local_rank, N.lib())
    ms_max = max_over_ranks(ms, world, dev)
    t_step = ms_max / args.steps * 1e-3
    # e2e through the public API on host numpy operands (H2D + product + D2H per call)
    e2e = None
    if st["api"] is not None and not args.no_e2e:
        Ah, Bh = st["host_ops"]()[:2]
        st["api"](Ah, Bh)
        e2e_steps = max(3, min(args.steps, 10))
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        for _ in range(e2e_steps):
            Mh, _ = st["api"](Ah, Bh)
        te = max_over_ranks(time.perf_counter() - t0, world, dev)
        e2e = {"value": job_throughput(e2e_steps, world, te), "unit": "products/s",
               "h2d_bytes_per_step": Ah.nbytes + Bh.nbytes, "d2h_bytes_per_step": Mh.nbytes,
               "steps": e2e_steps, "ms_per_step": 1e3 * te / e2e_steps,
               "path": "public API (reference signature) on host numpy arrays, one product per call"}
    if rank != 0:
        return
    pk = pipe_peaks()
    hbm, hbm_kind = hbm_peak()
    if "flops" in st:
        peak = pk.get(st["peak_key"])
        ach = st["flops"] / t_step / 1e12
        roof = {"bound": st["bound"], "kernel": "whole product", "achieved": ach, "peak": peak,
                "unit": "TFLOP/s", "frac": ach / peak if peak else None, "traffic": None,
                "peak_kind": f"measured ({pk.get('source')})", "alg_flops_per_step": st["flops"]}
        if "bytes_alt" in st:
            roof["hbm_frac"] = st["bytes_alt"] / t_step / 1e9 / hbm
        if "lds_bytes" in st and pk.get("lds64_tbs"):
            roof["datapath"] = {"resource": "shared-memory load bandwidth",
                                "achieved_tbs": st["lds_bytes"] / t_step / 1e12, "peak_tbs": pk["lds64_tbs"],
                                "frac": st["lds_bytes"] / t_step / 1e12 / pk["lds64_tbs"]}
    else:
        ach = st["bytes"] / t_step / 1e9
        roof = {"bound": "hbm", "kernel": "whole product", "achieved": ach, "peak": hbm, "unit": "GB/s",
                "frac": ach / hbm, "traffic": None, "peak_kind": hbm_kind, "alg_bytes_per_step": st["bytes"]}
    roof["ncu_limiters"] = ncu_limiters(cfg)
    line = {"metric": METRIC, "value": job_throughput(args.steps * st["units"], world, ms_max * 1e-3),
            "unit": "products/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": ms_max / args.steps, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": st["dtype"], "data": "synthetic",
            "config": {"workload": WORKLOADS[cfg], "n": st["n"], "units_per_step": st["units"],
                       "parallelism": f"replicas x{world}", "note": st["note"]},
            "clocks": clocks, "e2e": e2e, "gpu_launches": int(launches), "roofline": roof}
    if st["host_ops"] is not None and world == 1 and not args.no_cpu_baseline:
        ops = st["host_ops"]()
        t_cpu, Mo, ro = cpu_product(cfg, ops)
        hi = host_info()
        line["cpu_baseline"] = {"value": 1.0 / t_cpu, "unit": "products/s", "cores": hi["cores"], "kind": "port",
                                "sample": "one full product by the oracle port, timed with perf_counter", "host": hi}
        Mg = st["dev_out"]().cpu().numpy()
        line["parity_vs_oracle"] = {"rel": float(np.linalg.norm(Mg - Mo) / np.linalg.norm(Mo)),
                                    "tol": 1e-10, "note": "first product of the step's batch"}
        if cfg == "c3":  # near-tie protocol: the oracle's own picks vs the GPU's (forced above)
            import oracle as O
            subs, worst = 0, 0.0
            for key, gsel in (("magnitudes_a", ops[2][0]), ("magnitudes_b", ops[2][1])):
                mags = ro[key]
                own = O.top_indices(mags, 16)
                for a, b in zip(sorted(set(gsel) - set(own)), sorted(set(own) - set(gsel))):
                    subs += 1
                    worst = max(worst, abs(mags[a] - mags[b]) / np.spacing(np.max(mags)))
            line["parity_vs_oracle"]["near_tie_substitutions"] = subs
            line["parity_vs_oracle"]["worst_tie_gap_ulps"] = worst
    print(json.dumps(line), flush=True)


def run_c5_rows(args, rank, world, local_rank):
    """C5 at 1 < N < 8: one cycle product per step sharded by rows (sharded.cycle_product_rows)."""
    import torch
    import torch.distributed as dist

    from paper_2504_19308_b200 import _native as N
    from paper_2504_19308_b200 import genmat as G
    from paper_2504_19308_b200 import sharded as S

    dev = torch.device("cuda", local_rank)
    torch.cuda.set_device(dev)
    n, k = 32768, 128
    A, _ = G.c5_operand(n, 128, 32, 1234, 0, dev)
    B, _ = G.c5_operand(n, 128, 32, 1234, 1, dev)
    r0, r1 = S.cycle_row_range(n, world, rank)
    A_rows = A[r0:r1].contiguous()
    del A
    torch.cuda.empty_cache()
    M_rows = torch.empty(r1 - r0, n, dtype=torch.float32, device=dev)
    group = dist.group.WORLD if world > 1 else None
    res = {}

    def step():
        res["r"] = S.cycle_product_rows(A_rows, r0, B, k, k, 1, group=group, out=M_rows)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    ms, launches, clocks = _timed_region(step, args.steps, world, dev, local_rank, N.lib())
    ms_max = max_over_ranks(ms, world, dev)
    sel = res["r"]["sel_a"].to(torch.int64)
    sels = [torch.empty_like(sel) for _ in range(world)]
    if world > 1:
        dist.all_gather(sels, sel)
    else:
        sels = [sel]
    if rank == 0:
        pk = pipe_peaks()
        t_step = ms_max / args.steps * 1e-3
        flops = 4.0 * k * n * n
        line = {"metric": METRIC, "value": args.steps / (ms_max * 1e-3), "unit": "products/s", "n_gpus": world,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_max / args.steps,
                "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32",
                "data": "synthetic",
                "config": {"workload": WORKLOADS["c5"], "n": n,
                           "parallelism": f"rows x{world} (one product per step; all-gather + rank-order sum of "
                                          "A's cycle-energy partials and ||M_g||^2)"},
                "clocks": clocks, "e2e": None, "gpu_launches": int(launches),
                "roofline": {"bound": "fp32 (FFMA) / shared-memory datapath", "kernel": "whole product",
                             "achieved": flops / t_step / 1e12 / world, "peak": pk.get("fp32_ffma2_tflops"),
                             "unit": "TFLOP/s per GPU", "frac": (flops / t_step / 1e12 / world) / pk["fp32_ffma2_tflops"]
                             if pk.get("fp32_ffma2_tflops") else None, "traffic": None},
                "selection_equal_across_ranks": all(torch.equal(x, sels[0]) for x in sels)}
        print(json.dumps(line), flush=True)


# ------------------------------------------------------------------------------------------
# reference arm: the reference's CPU algorithm (oracle port), rank 0, full products
# ------------------------------------------------------------------------------------------
def run_reference(args, rank):
    if rank != 0:
        return
    import torch
    cfg = args.config
    hi = host_info()
    dev = torch.device("cuda", 0) if torch.cuda.is_available() else torch.device("cpu")
    if cfg == "c4":
        n = args.n
        A, B = gen_c4(n, 1234, dev)
        ops = (A.double().cpu().numpy(), B.double().cpu().numpy())
        del A, B

        def one():
            return cpu_c4_product(ops[0], ops[1], 7)[0]

        sample = f"one full n={n} C4 product per step (rSVD + cycle decomposition + all {n} rows)"
        dtype = "f64"
    elif cfg in ("c1", "c2", "c3"):
        st = _secondary_setup(cfg, 0, 1, dev)
        ops = st["host_ops"]()

        def one():
            return cpu_product(cfg, ops)[0]

        sample = f"one full {WORKLOADS[cfg]} per step"
        dtype = "f64"
    else:
        print(json.dumps({"impl": "reference", "unavailable": f"{cfg}: the full CPU product does not fit host "
                          "memory at n=32768 (parity uses oracle row samples, tests/test_gpu_c5*.py)"}))
        return
    for _ in range(min(args.warmup, 1)):
        one()
    times = [one() for _ in range(args.steps)]
    t = sum(times)
    v = args.steps / t
    line = {"metric": METRIC, "value": v, "unit": "products/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": min(args.warmup, 1), "ms_per_step": 1e3 * t / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": dtype,
            "data": "synthetic", "impl": "reference",
            "config": {"workload": WORKLOADS[cfg]},
            "cpu_baseline": {"value": v, "unit": "products/s", "cores": hi["cores"], "kind": "port",
                             "sample": sample + f"; median {1e3 * statistics.median(times):.0f} ms", "host": hi},
            "e2e": {"value": v, "unit": "products/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c4", choices=sorted(WORKLOADS))
    ap.add_argument("--n", type=int, default=N_DEFAULT)
    ap.add_argument("--plan", default="resid", choices=["resid", "direct"],
                    help="C4: residual plan (f16 gather over dA, default) or the all-fp32 gather over A")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--shard", default="auto", choices=["auto", "replicas", "rows"],
                    help="auto: c4 rows-sharded for N > 1 (BASELINE config 4), c5 rows for 1 < N < 8 "
                         "and one product per GPU at N = 8, replicas otherwise")
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
    shard = args.shard
    if shard == "auto":
        shard = ("rows" if (args.config == "c4" and world > 1) or (args.config == "c5" and 1 < world < 8)
                 else "replicas")
    try:
        if args.config == "c4":
            (run_c4_rows if shard == "rows" else run_c4)(args, rank, world, local_rank)
        elif args.config == "c5" and shard == "rows":
            run_c5_rows(args, rank, world, local_rank)
        else:
            run_secondary(args, rank, world, local_rank)
    finally:
        if world > 1:
            import torch.distributed as dist
            dist.destroy_process_group()


if __name__ == "__main__":
    main()
