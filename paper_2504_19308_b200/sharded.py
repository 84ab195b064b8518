"""Products sharded by rows of A and M over ranks: the C4 mixed product
(BASELINE config 4) and the cycle product (configs 2 and 5; ``cycle_rows_steps``, whose only
exchange before the product is the sum of the ranks' cycle-energy partials of A).

Rank g holds the row block A_g = A[r0:r1] and the whole B; it produces M[r0:r1]. The per-rank plan
is the single-device plan of apx_mixed_first_order (B's cycle decomposition and the persistent row
gather on one internal stream, the range finder on another) cut at the four points where rows
must be combined (apx_mixed_rows_phase, include/apx.h):

    Gram(Y_g) -> sum -> pass-1 Q_g, pass-2 Gram -> sum -> Bm_g = Q_g^T A_g -> sum -> W, M_g
              -> sum of [||A_g||^2, ||M_g||^2]

Only small factors cross ranks: two 64 x 64 fp64 Gram matrices, the 64 x n fp32 Bm (2 MiB at
n = 8192) and two scalars -- the "all-gather of the small truncated factors" of the north star.
Each exchange is an all-gather followed by a local sum in rank order (``ordered_sum``, SURVEY.md
§5 / §8(e)), never an NCCL all-reduce: the sum's bits then do not depend on the world size's
reduction tree or NCCL's algorithm choice, every rank holds the identical sum, and the result is
bitwise the lockstep (single-process) result. Every rank factors the same summed Gram, so the pass-2 decision and the
orthonormal basis agree across ranks; B's cycle selection is computed on every rank from the same
B (no exchange), so the selected indices are identical by construction.

``mixed_rows_steps`` is the rank-local generator (yields the tensor to sum at each exchange
point); ``mixed_product_rows`` drives it with torch.distributed (NCCL); ``lockstep`` drives
several shards inside one process, summing on the device in rank order (tests, single-GPU
simulation of the sharded math).
"""

from __future__ import annotations

import math

import torch

from . import _device as D
from . import _native as N


def row_range(n: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous row block [r0, r1) of rank `rank`: boundaries are r * n / world rounded to a
    multiple of 64 (the row-tile height of M += Q W), so every block is within 64 rows of n / world."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} of {world}")

    def cut(r):
        return n if r == world else min(n, 64 * round(r * n / (64 * world)))

    return cut(rank), cut(rank + 1)


def mixed_rows_steps(A_rows, B, k_svd: int, k_cyc: int, order: int, omega, out=None, serialize: bool = False):
    """One rank's share of the C4 product. A_rows (m x n), B (n x n), omega (n x k_svd): fp32 device
    tensors. Yields the tensor to be summed over ranks (in place) at each of the four exchange
    points; returns dict(M=rows of M, sel_b, scalars) with the scalars of apx_mixed_first_order.
    serialize: start M_g += Q_g W only after this shard's whole gather (required when several shards
    share one device, see apx_mixed_rows_phase)."""
    if A_rows.dtype != torch.float32 or B.dtype != torch.float32:
        raise ValueError("the sharded product is fp32")
    m, n = A_rows.shape
    if tuple(B.shape) != (n, n):
        raise ValueError(f"B must be {n} x {n}, got {tuple(B.shape)}")
    if order not in (0, 1):
        raise ValueError("order must be 0 or 1")
    dev = A_rows.device
    l = k_svd
    M = out if out is not None else torch.empty((m, n), dtype=torch.float32, device=dev)
    sb = torch.empty(max(k_cyc, 1), dtype=torch.int32, device=dev)
    scal = torch.zeros(N.NSCALARS, dtype=torch.float64, device=dev)
    ws = D.workspace(N.size("apx_mixed_rows_workspace", n, m, k_svd, k_cyc))
    g1 = torch.empty(l * l, dtype=torch.float64, device=dev)
    g2 = torch.empty(l * l, dtype=torch.float64, device=dev)
    bm = torch.empty(l * n, dtype=torch.float32, device=dev)
    fin = torch.zeros(3, dtype=torch.float64, device=dev)

    def phase(i, red_in, red_out):
        N.call("apx_mixed_rows_phase", i, A_rows.data_ptr(), m, B.data_ptr(), n, k_svd, k_cyc, order,
               1 if serialize else 0, omega.data_ptr(), M.data_ptr(), sb.data_ptr(), D.ptr(red_in),
               red_out.data_ptr(), scal.data_ptr(), ws.data_ptr(), ws.numel(), D.stream_ptr())

    phase(1, None, g1)
    yield g1
    phase(2, g1, g2)
    yield g2
    phase(3, g2, bm)
    yield bm
    phase(4, bm, fin)
    yield fin[:2]
    scal[N.S_FRO2_A] = fin[0]  # device-side copies: no host synchronisation inside the product
    scal[N.S_FRO2_M] = fin[1]
    return {"M": M, "sel_b": sb[:k_cyc], "scalars": scal, "breakdown": fin[2], "ws": ws}


def cycle_row_range(n: int, world: int, rank: int, align: int = 128) -> tuple[int, int]:
    """Row block of `rank` for the sharded cycle product: boundaries r * n / world rounded to a
    multiple of `align` (the column chunk of the large-n left product, 128 fp32 / 64 fp64)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} of {world}")

    def cut(r):
        return n if r == world else min(n, align * round(r * n / (align * world)))

    return cut(rank), cut(rank + 1)


def cycle_rows_steps(A_rows, row0: int, B, k_a: int, k_b: int, order: int, out=None):
    """One rank's share of the cycle product (C2 / C5 sharded by rows). A_rows
    (m x n, global rows row0..row0+m) and B (n x n): device tensors of one real dtype. Yields the
    tensor to be summed over ranks at each exchange point -- A's cycle energies over the rank's
    rows (n fp64), then [||M_g||^2] -- and returns dict(M=rows of M, sel_a, sel_b, scalars)."""
    m, n = A_rows.shape
    if tuple(B.shape) != (n, n) or B.dtype != A_rows.dtype:
        raise ValueError(f"B must be {n} x {n} of A's dtype, got {tuple(B.shape)} {B.dtype}")
    if order not in (0, 1):
        raise ValueError("order must be 0 or 1")
    if A_rows.dtype not in (torch.float32, torch.float64):
        raise ValueError("real fp32 / fp64 operands required")
    code = N.APX_F32 if A_rows.dtype == torch.float32 else N.APX_F64
    dev = A_rows.device
    M = out if out is not None else torch.empty((m, n), dtype=A_rows.dtype, device=dev)
    sa = torch.empty(max(k_a, 1), dtype=torch.int32, device=dev)
    sb = torch.empty(max(k_b, 1), dtype=torch.int32, device=dev)
    scal = torch.zeros(N.NSCALARS, dtype=torch.float64, device=dev)
    ws = D.workspace(N.size("apx_cycle_rows_workspace", code, n, m, k_a, k_b, order))
    energies = torch.empty(n, dtype=torch.float64, device=dev)
    fin = torch.zeros(1, dtype=torch.float64, device=dev)

    def phase(i, red_in, red_out):
        N.call("apx_cycle_rows_phase", i, code, A_rows.data_ptr(), m, row0, B.data_ptr(), n, k_a, k_b, order,
               M.data_ptr(), sa.data_ptr(), sb.data_ptr(), D.ptr(red_in), red_out.data_ptr(), scal.data_ptr(),
               ws.data_ptr(), ws.numel(), D.stream_ptr())

    phase(1, None, energies)
    yield energies
    phase(2, energies, fin)
    yield fin
    scal[N.S_FRO2_M] = fin[0]
    return {"M": M, "sel_a": sa[:k_a], "sel_b": sb[:k_b], "scalars": scal, "ws": ws}


def cycle_product_rows(A_rows, row0: int, B, k_a: int, k_b: int, order: int, group=None, out=None):
    """This rank's rows of the cycle product; the two exchanges are ordered all-gather sums
    (``ordered_sum``: NCCL on the current stream for CUDA tensors)."""
    return _drive(cycle_rows_steps(A_rows, row0, B, k_a, k_b, order, out), lambda t: ordered_sum(t, group))


def rank_order_sum(parts):
    """Sum of the per-rank tensors in rank order: ((p0 + p1) + p2) + ... (the order lockstep uses)."""
    total = parts[0].clone()
    for t in parts[1:]:
        total += t
    return total


def ordered_sum(t, group=None):
    """In place: t <- sum over ranks of t, as an all-gather plus a fixed rank-order local sum
    (deterministic and identical on every rank, independent of NCCL's reduction algorithm).
    NCCL groups gather into one buffer (ncclAllGather); other backends (gloo) gather a list."""
    import torch.distributed as dist

    # no process group: a single-process run is a world of one (bench.py --gpus 1 --shard rows)
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    if world == 1:
        return t
    flat = t.contiguous().view(-1)
    if dist.get_backend(group) == "nccl":
        buf = torch.empty((world, flat.numel()), dtype=t.dtype, device=t.device)
        dist.all_gather_into_tensor(buf, flat, group=group)
        parts = list(buf.unbind(0))
    else:
        parts = [torch.empty_like(flat) for _ in range(world)]
        dist.all_gather(parts, flat, group=group)
    t.view(-1).copy_(rank_order_sum(parts))
    return t


def check_breakdown(result):
    """Raise if the row-sharded CholeskyQR broke down (reads one device scalar)."""
    if float(result["breakdown"].item()) != 0.0:
        raise RuntimeError("row-sharded CholeskyQR broke down (numerically rank-deficient sketch); "
                           "use the single-device product, whose Householder fallback handles it")
    return result


def _drive(gen, reduce):
    try:
        t = next(gen)
        while True:
            reduce(t)
            t = gen.send(None)
    except StopIteration as e:
        return e.value


def mixed_product_rows(A_rows, B, k_svd: int, k_cyc: int, order: int, omega, group=None, out=None,
                       check: bool = True):
    """This rank's rows of the C4 product; the exchanges are ordered all-gather sums
    (``ordered_sum``: NCCL on the current stream for CUDA tensors). check=False skips the
    (synchronising) breakdown check -- call check_breakdown(result) later."""
    r = _drive(mixed_rows_steps(A_rows, B, k_svd, k_cyc, order, omega, out), lambda t: ordered_sum(t, group))
    return check_breakdown(r) if check else r


def lockstep(gens):
    """Run the generators of several shards in one process: at every exchange point the yielded
    tensors are summed in rank order on the device and the sum is written back into each (what
    an all-reduce does across processes). Returns the list of results. The shards must have been
    created with serialize=True when they share a device."""
    pending = [next(g) for g in gens]
    results = [None] * len(gens)
    while True:
        total = rank_order_sum(pending)
        nxt = []
        for i, (g, t) in enumerate(zip(gens, pending)):
            t.copy_(total)
            try:
                nxt.append(g.send(None))
            except StopIteration as e:
                results[i] = e.value
                nxt.append(None)
        if all(r is not None for r in results):
            return results
        if any(x is None for x in nxt):
            raise RuntimeError("shards disagree on the number of exchange points")
        pending = nxt


def norms_from_scalars(s, n: int):
    """(||A||, ||B||, ||dA||, ||dB||, ||M||) of an n x n product from the scalar vector."""
    from .cycle import _norms

    return _norms(s, n * n)


# ---- the circulant product sharded by rows of M (C3 / C5-secondary) -----------
# term1 = Ahat B is column-local (circulant.py:136-147), term2 = dA Bhat row-local (:150-161): a
# rank computes term1 for a block of COLUMNS and term2 for its block of ROWS, and one all-to-all
# moves term1's pieces to the ranks that own their rows. The decompositions are split by cycle
# blocks (zero-padded partial magnitudes and selected spectra, summed = gathered in rank order),
# so selections and every row of M are bitwise the single-device product's.

def _even_cut(n: int, world: int, r: int) -> int:
    return n if r == world else min(n, 2 * round(r * n / (2 * world)))


def circulant_partition(n: int, world: int, rank: int):
    """(rows, cols, cycle blocks) of `rank`: rows and columns [r0, r1) cut at even indices (the
    kernels pair rows / columns), cycle blocks an even split of the decomposition grid."""
    import ctypes as C

    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} of {world}")
    parts, cpc = C.c_int64(), C.c_int64()
    N.call("apx_circulant_rows_grid", n, C.addressof(parts), C.addressof(cpc))
    P = parts.value
    rows = (_even_cut(n, world, rank), _even_cut(n, world, rank + 1))
    blks = (round(rank * P / world), round((rank + 1) * P / world))
    return rows, rows, blks, P


def circulant_rows_steps(A, B, k: int, order: int, world: int, rank: int, out=None):
    """One rank's share of the circulant product on replicated device operands A, B (n x n fp64 or
    complex128). Yields ("sum", t) at the three summing exchanges and ("rows", T1, M_rows, plan) at
    the all-to-all (plan = every rank's (rows, cols)); returns dict(M=rows of M (complex128),
    sel_a, sel_b, scalars, rows)."""
    n = A.shape[0]
    if tuple(A.shape) != (n, n) or tuple(B.shape) != (n, n):
        raise ValueError("two square n x n operands required")
    if order not in (0, 1):
        raise ValueError("order must be 0 or 1")
    cplx = A.is_complex() or B.is_complex()
    code = N.APX_C128 if cplx else N.APX_F64
    dt = torch.complex128 if cplx else torch.float64
    A, B = A.to(dt).contiguous(), B.to(dt).contiguous()
    dev = A.device
    (r0, r1), (c0, c1), (b0, b1), P = circulant_partition(n, world, rank)
    plan = [circulant_partition(n, world, h)[:2] for h in range(world)]
    m, w = r1 - r0, c1 - c0
    M = out if out is not None else torch.zeros((m, n), dtype=torch.complex128, device=dev)
    T1 = torch.empty((n, max(w, 1)), dtype=torch.complex128, device=dev)
    sa = torch.empty(max(k, 1), dtype=torch.int32, device=dev)
    sb = torch.empty(max(k, 1), dtype=torch.int32, device=dev)
    scal = torch.zeros(N.NSCALARS, dtype=torch.float64, device=dev)
    ws = D.workspace(N.size("apx_circulant_rows_workspace", code, n, k, m, b0, b1))
    red1 = torch.zeros(2 * P * n, dtype=torch.float64, device=dev)
    red2 = torch.zeros(2 * max(k, 1) * n, dtype=torch.complex128, device=dev)
    fin = torch.zeros(1, dtype=torch.float64, device=dev)

    def phase(i, red_in, red_out):
        N.call("apx_circulant_rows_phase", i, code, A.data_ptr(), B.data_ptr(), n, k, order, r0, m, c0, w, b0, b1,
               M.data_ptr(), T1.data_ptr(), sa.data_ptr(), sb.data_ptr(), D.ptr(red_in), D.ptr(red_out),
               scal.data_ptr(), ws.data_ptr(), ws.numel(), D.stream_ptr())

    phase(1, None, red1)
    yield ("sum", red1)
    phase(2, red1, red2)
    yield ("sum", red2.view(torch.float64))
    phase(3, red2, None)
    yield ("rows", T1[:, :w], M, plan)
    phase(4, None, fin)
    yield ("sum", fin)
    scal[N.S_FRO2_M] = fin[0]
    return {"M": M, "sel_a": sa[:k], "sel_b": sb[:k], "scalars": scal, "rows": (r0, r1), "ws": ws}


def _a2a_rows(T1, M_rows, plan, rank, group=None):
    """All-to-all of term1's pieces: rank g sends T1[rows of h, :] (its columns) to every h and
    places what it receives at M_rows[:, cols of h]."""
    import torch.distributed as dist

    (r0, r1), _ = plan[rank]
    m = r1 - r0
    w = T1.shape[1]
    send = torch.cat([T1[a:b].reshape(-1) for (a, b), _ in plan]) if w else T1.new_zeros(0)
    in_splits = [(b - a) * w for (a, b), _ in plan]
    out_splits = [m * (d - c) for _, (c, d) in plan]
    recv = torch.empty(sum(out_splits), dtype=T1.dtype, device=T1.device)
    if not dist.is_initialized():  # a world of one: the piece stays
        recv.copy_(send)
    elif dist.get_backend(group) == "nccl":
        dist.all_to_all_single(torch.view_as_real(recv).view(-1), torch.view_as_real(send).view(-1),
                               [2 * x for x in out_splits], [2 * x for x in in_splits], group=group)
    else:  # gloo has no alltoall: pairwise point-to-point exchanges (the grouped send/recv form)
        outs = list(recv.split(out_splits))
        ins = list(send.split(in_splits))
        outs[rank].copy_(ins[rank])
        reqs = []
        for h in range(len(plan)):
            if h != rank:
                reqs.append(dist.isend(ins[h].contiguous(), dist.get_global_rank(group, h) if group else h, group=group))
                reqs.append(dist.irecv(outs[h], dist.get_global_rank(group, h) if group else h, group=group))
        for r in reqs:
            r.wait()
        recv = torch.cat(outs)
    off = 0
    for (_, (c, d)), sz in zip(plan, out_splits):
        M_rows[:, c:d] = recv[off:off + sz].view(m, d - c)
        off += sz


def circulant_product_rows(A, B, k: int, order: int, group=None, out=None):
    """This rank's rows of the circulant product (the exchanges over torch.distributed)."""
    import torch.distributed as dist

    world, rank = (dist.get_world_size(group), dist.get_rank(group)) if dist.is_initialized() else (1, 0)
    gen = circulant_rows_steps(A, B, k, order, world, rank, out)
    try:
        req = next(gen)
        while True:
            if req[0] == "sum":
                ordered_sum(req[1], group)
            else:
                _a2a_rows(req[1], req[2], req[3], rank, group)
            req = gen.send(None)
    except StopIteration as e:
        return e.value


def circulant_lockstep(gens):
    """Drive the circulant shards of one process (tests; single-GPU simulation): rank-order sums
    at the summing exchanges, the term1 redistribution done by slicing."""
    reqs = [next(g) for g in gens]
    results = [None] * len(gens)
    while True:
        kind = reqs[0][0]
        if any(r[0] != kind for r in reqs):
            raise RuntimeError("shards disagree on the exchange sequence")
        if kind == "sum":
            total = rank_order_sum([r[1] for r in reqs])
            for r in reqs:
                r[1].copy_(total)
        else:
            plan = reqs[0][3]
            for g, r in enumerate(reqs):
                (a, b), _ = plan[g]
                for h, rh in enumerate(reqs):
                    _, (c, d) = plan[h]
                    r[2][:, c:d] = rh[1][a:b]
        nxt = []
        for i, g in enumerate(gens):
            try:
                nxt.append(g.send(None))
            except StopIteration as e:
                results[i] = e.value
                nxt.append(None)
        if all(x is not None for x in results):
            return results
        if any(x is None for x in nxt):
            raise RuntimeError("shards disagree on the number of exchange points")
        reqs = nxt


# ---- the sfft product sharded by rows (fsparse.py:168-240; SURVEY.md §8(e) secondary) ------------
# Rows of At = A W* and A's per-row selection are row-local; B is replicated, so Bt = W B, its
# selection and SB are the same on every rank. The only exchange: [||A_g||^2, ||dAt_g||^2,
# ||M_g||^2].

def sfft_rows_steps(A_rows, B, k: int, order: int, sparsify_b: str = "rows", out=None):
    """One rank's rows of the sfft product (device operands, fp64 or complex128). Yields the
    3-vector to sum over ranks; returns dict(M=rows of M, sel_a (rank rows), sel_b, scalars)."""
    from .fsparse import sfft_product_device

    if sparsify_b not in ("rows", "cols"):
        raise ValueError(f"unknown sparsify_b {sparsify_b!r}")
    cplx = A_rows.is_complex() or B.is_complex()
    code = N.APX_C128 if cplx else N.APX_F64
    dt = torch.complex128 if cplx else torch.float64
    r = sfft_product_device(A_rows.to(dt).contiguous(), B.to(dt).contiguous(), code, k, order,
                            sparsify_b == "cols", out)
    s = r["scalars"]
    part = torch.stack([s[N.S_FRO2_A], s[N.S_RES2_A], s[N.S_FRO2_M]])
    yield part
    s[N.S_FRO2_A], s[N.S_RES2_A], s[N.S_FRO2_M] = part[0], part[1], part[2]
    return r


def sfft_product_rows(A_rows, B, k: int, order: int, sparsify_b: str = "rows", group=None, out=None):
    """This rank's rows of the sfft product (one ordered-sum exchange over torch.distributed)."""
    return _drive(sfft_rows_steps(A_rows, B, k, order, sparsify_b, out), lambda t: ordered_sum(t, group))
