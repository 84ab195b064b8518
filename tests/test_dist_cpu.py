"""The N > 1 path on CPU: world_size-2 gloo process group over 127.0.0.1 (bench.py's replica
plumbing -- independent products per rank, max-over-ranks job time, whole-job throughput)."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, times, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import bench
        ms_max = bench.max_over_ranks(times[rank], world, torch.device("cpu"))
        value = bench.job_throughput(5, world, ms_max * 1e-3)
        seeds = [None] * world
        dist.all_gather_object(seeds, bench.replica_seed(rank))
        q.put((rank, ms_max, value, seeds))
    finally:
        dist.destroy_process_group()


def test_two_rank_replicas_gloo():
    world, port = 2, _free_port()
    times = [12.5, 17.25]  # per-rank device ms for 5 steps
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, times, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, ms_max, value, seeds in out:
        assert ms_max == max(times)                      # slowest rank sets the job time
        assert value == pytest.approx(world * 5 / (max(times) * 1e-3))
        assert len(set(seeds)) == world                  # independent replica inputs


def test_single_rank_no_collective():
    import bench
    assert bench.max_over_ranks(3.5, 1, torch.device("cpu")) == 3.5
    assert bench.job_throughput(4, 1, 2.0) == 2.0


# ---- the row-sharded product's exchange protocol (paper_2504_19308_b200.sharded) over gloo ----
# The device phases are replaced by their fp64 algebra on CPU tensors (test-only stand-ins); what
# is checked is the host protocol the GPU path uses -- one in-place ordered sum per exchange point,
# in order -- and that the row-block algebra reproduces the unsharded projection Q Q^T A.

def _toy_rows_steps(A_rows, Omega):
    Y = A_rows @ Omega
    G = Y.T @ Y
    yield G                                   # Gram partial -> sum over ranks
    R = torch.linalg.cholesky(G).T            # upper factor, identical on every rank
    Q = torch.linalg.solve_triangular(R, Y, upper=True, left=False)
    Bm = Q.T @ A_rows
    yield Bm                                  # Q_g^T A_g -> sum over ranks
    return Q @ Bm                             # rows of Q Q^T A


def _sharded_worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2504_19308_b200.sharded import _drive, ordered_sum, row_range
        g = torch.Generator().manual_seed(7)
        n, l = 320, 8
        A = torch.randn(n, n, generator=g, dtype=torch.float64)
        Omega = torch.randn(n, l, generator=g, dtype=torch.float64)
        r0, r1 = row_range(n, world, rank)
        P_rows = _drive(_toy_rows_steps(A[r0:r1], Omega), ordered_sum)
        q.put((rank, r0, r1, P_rows.numpy()))
    finally:
        dist.destroy_process_group()


def test_row_sharded_protocol_gloo():
    import numpy as np
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_sharded_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = sorted(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    g = torch.Generator().manual_seed(7)
    n, l = 320, 8
    A = torch.randn(n, n, generator=g, dtype=torch.float64)
    Omega = torch.randn(n, l, generator=g, dtype=torch.float64)
    Qf, _ = torch.linalg.qr(A @ Omega)
    P = (Qf @ (Qf.T @ A)).numpy()
    got = np.concatenate([o[3] for o in out], axis=0)
    assert [o[1:3] for o in out] == [(0, 128), (128, 320)]
    assert np.linalg.norm(got - P) <= 1e-10 * np.linalg.norm(P)


def test_row_range_partition():
    from paper_2504_19308_b200.sharded import row_range
    for n in (128, 1000, 8192, 32768):
        for world in (1, 2, 3, 4, 8):
            blocks = [row_range(n, world, r) for r in range(world)]
            assert blocks[0][0] == 0 and blocks[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(blocks, blocks[1:]))
            sizes = [b - a for a, b in blocks]
            assert all(abs(z - n / world) <= 64 for z in sizes)
    with pytest.raises(ValueError):
        row_range(128, 2, 2)


# ---- the row-sharded cycle product's protocol (sharded.cycle_rows_steps) over gloo ----
# Device phases replaced by the oracle restatement on CPU (test-only stand-ins): the rank's cycle
# energy partials -> all-reduce -> selection from the summed energies -> the rank's product rows
# (oracle.cycle_product_rows) -> all-reduce of ||M_g||^2. The concatenated rows must equal the
# unsharded oracle product, and every rank must select the same cycles.

def _toy_cycle_rows_steps(A, B, r0, r1, k):
    import numpy as np
    import oracle as O
    n = A.shape[0]
    i = np.arange(r0, r1)
    e = torch.zeros(n, dtype=torch.float64)
    for j in range(n):
        e[j] = float(np.sum(A[i, (i - j) % n] ** 2))
    yield e                                            # energy partials -> sum over ranks
    JA = O.top_indices(np.sqrt(e.numpy()), k)
    JB, lamB, _, _, _ = O.cycle_decompose(B, k)
    rows = np.arange(r0, r1)
    Mg = O.cycle_product_rows(rows, A[rows], JA, [B[(rows - j) % n] for j in JA], JB, lamB)
    fin = torch.tensor([float(np.sum(Mg ** 2))], dtype=torch.float64)
    yield fin                                          # ||M_g||^2 -> sum over ranks
    return JA, Mg, float(fin[0])


def _sharded_cycle_worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle as O
        from paper_2504_19308_b200.sharded import _drive, cycle_row_range, ordered_sum
        n, k = 256, 8
        A, B = O.gen_cycle_operand(n, k, 31), O.gen_cycle_operand(n, k, 32)
        r0, r1 = cycle_row_range(n, world, rank, align=64)
        JA, Mg, fro2 = _drive(_toy_cycle_rows_steps(A, B, r0, r1, k), ordered_sum)
        q.put((rank, r0, r1, JA, Mg, fro2))
    finally:
        dist.destroy_process_group()


def test_row_sharded_cycle_protocol_gloo():
    import numpy as np
    import oracle as O
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_sharded_cycle_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = sorted((q.get(timeout=120) for _ in range(world)), key=lambda o: o[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    n, k = 256, 8
    A, B = O.gen_cycle_operand(n, k, 31), O.gen_cycle_operand(n, k, 32)
    M, rep = O.cycle_first_order_multiply(A, B, k, 1)
    assert [o[1:3] for o in out] == [(0, 128), (128, 256)]
    assert out[0][3] == out[1][3] == rep["selected_a"]
    got = np.concatenate([o[4] for o in out], axis=0)
    assert np.linalg.norm(got - M) <= 1e-12 * np.linalg.norm(M)
    assert out[0][5] == out[1][5] == pytest.approx(float(np.sum(M ** 2)), rel=1e-12)


def test_cycle_row_range_partition():
    from paper_2504_19308_b200.sharded import cycle_row_range
    for n, align in ((2048, 64), (16384, 128), (32768, 128)):
        for world in (1, 2, 3, 4, 8):
            blocks = [cycle_row_range(n, world, r, align) for r in range(world)]
            assert blocks[0][0] == 0 and blocks[-1][1] == n
            assert all(a[1] == b[0] and a[0] % align == 0 for a, b in zip(blocks, blocks[1:]))


# ---- ordered_sum: all-gather + rank-order sum, bitwise equal on every rank ----

def _ordered_worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2504_19308_b200.sharded import ordered_sum
        g = torch.Generator().manual_seed(100 + rank)
        # magnitudes spread over 1e-8..1e8: a different summation order changes the last bits
        t = torch.randn(4096, generator=g, dtype=torch.float64) * torch.logspace(-8, 8, 4096, dtype=torch.float64)
        t32 = t.float().reshape(64, 64)
        ordered_sum(t)
        ordered_sum(t32)
        q.put((rank, t.numpy().tobytes(), t32.numpy().tobytes()))
    finally:
        dist.destroy_process_group()


def test_ordered_sum_bitwise_gloo():
    import numpy as np
    from paper_2504_19308_b200.sharded import rank_order_sum
    world, port = 3, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_ordered_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = sorted((q.get(timeout=120) for _ in range(world)), key=lambda o: o[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    parts = []
    for r in range(world):
        g = torch.Generator().manual_seed(100 + r)
        parts.append(torch.randn(4096, generator=g, dtype=torch.float64) *
                     torch.logspace(-8, 8, 4096, dtype=torch.float64))
    want = rank_order_sum(parts).numpy().tobytes()
    want32 = rank_order_sum([p.float().reshape(64, 64) for p in parts]).numpy().tobytes()
    assert all(o[1] == want for o in out)          # identical bits on every rank = lockstep's order
    assert all(o[2] == want32 for o in out)


# ---- the row-sharded circulant product's protocol (sharded.circulant_rows_steps) over gloo ----
# Device phases replaced by the oracle on CPU (test-only stand-ins): magnitude partials of the
# rank's cycles -> ordered sum -> selection; selected spectrum rows of the rank's cycles
# (zero-padded) -> ordered sum; term1 for the rank's COLUMNS -> all-to-all (sharded._a2a_rows,
# the function the GPU path uses) into the rank's rows; term2 for the rank's ROWS; ||M_g||^2 -> sum.

def _toy_circ_rows_steps(A, B, k, world, rank):
    import numpy as np
    import oracle as O
    from oracle import apx_oracle as OX
    n = A.shape[0]
    a0, a1 = (rank * n) // world, ((rank + 1) * n) // world        # cycle block of this rank
    r0, r1 = 2 * round(rank * n / (2 * world)), n if rank == world - 1 else 2 * round((rank + 1) * n / (2 * world))
    plan = []
    for h in range(world):
        h0 = 2 * round(h * n / (2 * world))
        h1 = n if h == world - 1 else 2 * round((h + 1) * n / (2 * world))
        plan.append(((h0, h1), (h0, h1)))
    Sa, _ = O.circulant_decompose(A)
    Sb, _ = O.circulant_decompose(B)
    part = torch.zeros(2, n, dtype=torch.float64)
    part[0] = torch.from_numpy(np.sum(np.abs(Sa[:, a0:a1]) ** 2, axis=1))
    part[1] = torch.from_numpy(np.sum(np.abs(Sb[:, a0:a1]) ** 2, axis=1))
    yield ("sum", part)
    sel_a = O.top_indices(np.sqrt(part[0].numpy()), k)
    sel_b = O.top_indices(np.sqrt(part[1].numpy()), k)
    spec = torch.zeros(2, n, n, dtype=torch.complex128)   # rows t of S from this rank's cycles j
    spec[0][:, a0:a1] = torch.from_numpy(Sa[:, a0:a1])
    spec[1][:, a0:a1] = torch.from_numpy(Sb[:, a0:a1])
    yield ("sum", torch.view_as_real(spec))
    Sa_g, Sb_g = spec[0].numpy(), spec[1].numpy()
    c0, c1 = plan[rank][1]
    FB = OX.unitary_dft(B, "forward", axis=0)
    T1 = torch.from_numpy(np.ascontiguousarray(O.circulant_left_product(Sa_g, sel_a, FB[:, c0:c1])))
    M = torch.zeros(r1 - r0, n, dtype=torch.complex128)
    yield ("rows", T1, M, plan)
    dA = A[r0:r1] - O.circulant_materialize(Sa_g, sel_a)[r0:r1]
    M += torch.from_numpy(O.circulant_right_product(Sb_g, sel_b, dA))
    fin = torch.tensor([float(torch.sum(torch.abs(M) ** 2))], dtype=torch.float64)
    yield ("sum", fin)
    return (r0, r1), sel_a, sel_b, M.numpy(), float(fin[0])


def _sharded_circ_worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle as O
        from paper_2504_19308_b200.sharded import _a2a_rows, ordered_sum
        n, k = 64, 6
        A, B = O.gen_circulant_operand(n, 4, 41), O.gen_circulant_operand(n, 4, 42)
        gen = _toy_circ_rows_steps(A, B, k, world, rank)
        req = next(gen)
        try:
            while True:
                if req[0] == "sum":
                    ordered_sum(req[1])
                else:
                    _a2a_rows(req[1], req[2], req[3], rank)
                req = gen.send(None)
        except StopIteration as e:
            q.put((rank,) + e.value)
    finally:
        dist.destroy_process_group()


def test_row_sharded_circulant_protocol_gloo():
    import numpy as np
    import oracle as O
    world, port = 3, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_sharded_circ_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = sorted((q.get(timeout=120) for _ in range(world)), key=lambda o: o[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    n, k = 64, 6
    A, B = O.gen_circulant_operand(n, 4, 41), O.gen_circulant_operand(n, 4, 42)
    sel_a = [o[2] for o in out]
    M, rep = O.circulant_first_order_multiply(A, B, k, 1, sel_a[0], out[0][3])
    assert all(s == sel_a[0] for s in sel_a)                   # one selection on every rank
    got = np.concatenate([o[4] for o in out], axis=0)
    assert [o[1] for o in out] == [(0, 22), (22, 42), (42, 64)]
    assert np.linalg.norm(got - M) <= 1e-12 * np.linalg.norm(M)
    assert out[0][5] == pytest.approx(float(np.sum(np.abs(M) ** 2)), rel=1e-12)


# ---- the row-sharded sfft product (sharded.sfft_rows_steps): rows of the oracle's product are
# row-local, so each rank's oracle product on its rows of A is those rows of the full product ----

def _sharded_sfft_worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import numpy as np
        import oracle as O
        from paper_2504_19308_b200.sharded import ordered_sum
        rng = np.random.default_rng(9)
        A, B = rng.standard_normal((40, 32)), rng.standard_normal((32, 24))
        r0, r1 = (rank * 40) // world, ((rank + 1) * 40) // world
        Mg, rep = O.fft_sparse_first_order_multiply(A[r0:r1], B, 5, 1, "rows")
        part = torch.tensor([float(np.sum(A[r0:r1] ** 2)), rep["norm_da"] ** 2, float(np.sum(np.abs(Mg) ** 2))],
                            dtype=torch.float64)
        ordered_sum(part)
        q.put((rank, Mg, part.numpy()))
    finally:
        dist.destroy_process_group()


def test_row_sharded_sfft_protocol_gloo():
    import numpy as np
    import oracle as O
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_sharded_sfft_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = sorted((q.get(timeout=120) for _ in range(world)), key=lambda o: o[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    rng = np.random.default_rng(9)
    A, B = rng.standard_normal((40, 32)), rng.standard_normal((32, 24))
    M, rep = O.fft_sparse_first_order_multiply(A, B, 5, 1, "rows")
    got = np.concatenate([o[1] for o in out], axis=0)
    assert np.linalg.norm(got - M) <= 1e-12 * np.linalg.norm(M)
    fro2, res2, m2 = out[0][2]
    assert fro2 == pytest.approx(float(np.sum(A ** 2)), rel=1e-12)
    assert res2 == pytest.approx(rep["norm_da"] ** 2, rel=1e-12)
    assert m2 == pytest.approx(float(np.sum(np.abs(M) ** 2)), rel=1e-12)


def test_ordered_sum_without_process_group_is_identity():
    """A single-process run (no torch.distributed group) is a world of one: ordered_sum returns its
    argument untouched instead of raising (bench.py --gpus 1 --shard rows)."""
    import torch
    import torch.distributed as dist
    from paper_2504_19308_b200 import sharded as S

    assert not dist.is_initialized()
    t = torch.arange(6, dtype=torch.float64).reshape(2, 3)
    ref = t.clone()
    assert S.ordered_sum(t) is t
    assert torch.equal(t, ref)
