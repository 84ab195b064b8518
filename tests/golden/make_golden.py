"""Generate the golden vectors that pin the oracle (and, through it, the GPU path).

Run ONCE in the build container, where the reference is importable:

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

It imports the unmodified reference package from /root/reference/pkg/src and records its own
outputs on small seeded inputs into tests/golden/*.npz. Nothing at test time reads
/root/reference: the fixtures travel with the repo.

The cycle and mixed products are not reference functions; their fixtures are composed here from
the reference's own primitives (cycle_reorder / cycle_reorder_inverse / apply_cycle_power /
top_indices / randomized_partial_svd), so the restated oracle is pinned against those.
"""

from __future__ import annotations

import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
sys.path.insert(0, REF)
sys.dont_write_bytecode = True

import apxmm  # noqa: E402
from apxmm import circulant as rc  # noqa: E402
from apxmm import core as rcore  # noqa: E402
from apxmm import fsparse as rf  # noqa: E402
from apxmm import svd as rs  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def rep_arr(rep):
    return np.array([rep.norm_da, rep.norm_db,
                     np.nan if rep.apriori_estimate is None else rep.apriori_estimate,
                     np.nan if rep.posterior_estimate is None else rep.posterior_estimate,
                     rep.k], dtype=float)


def core_cases():
    d = {}
    A4 = np.arange(16.0).reshape(4, 4)
    d["cr_A4"] = A4
    d["cr_right_A4"] = rcore.cycle_reorder(A4, "right")
    d["cr_left_A4"] = rcore.cycle_reorder(A4, "left")
    rng = np.random.default_rng(100)
    for n in (1, 5, 7, 33):
        A = rng.standard_normal((n, n))
        d[f"cr_A{n}r"] = A
        d[f"cr_right_A{n}r"] = rcore.cycle_reorder(A, "right")
        d[f"cr_left_A{n}r"] = rcore.cycle_reorder(A, "left")
    M = rng.standard_normal((6, 6))
    d["acp_M"] = M
    for kk in (0, 1, 5):
        d[f"acp_left_{kk}"] = rcore.apply_cycle_power(M, kk, "left")
        d[f"acp_right_{kk}"] = rcore.apply_cycle_power(M, kk, "right")
    for n in (1, 2, 3, 4, 5, 7, 8, 16, 31, 64, 97, 128, 700):
        x = rng.standard_normal((n, 3)) + 1j * rng.standard_normal((n, 3))
        d[f"dft_x{n}"] = x
        d[f"dft_fwd{n}"] = rcore.unitary_dft(x, "forward", axis=0)
        d[f"dft_inv{n}"] = rcore.unitary_dft(x, "inverse", axis=0)
    w = np.array([1.0, 3.0, 3.0, 2.0, 0.0, 3.0, 2.0, 2.0])
    d["ti_w"] = w
    for kk in range(0, 9):
        d[f"ti_{kk}"] = np.array(rc.top_indices(w, kk), dtype=np.int64)
    np.savez_compressed(os.path.join(OUT, "core.npz"), **d)


def circulant_cases():
    d = {}
    rng = np.random.default_rng(200)
    cases = [(2, 1), (8, 3), (16, 6), (31, 6), (32, 6), (64, 8), (97, 5)]
    for n, k in cases:
        A = rng.standard_normal((n, n))
        B = rng.standard_normal((n, n))
        d[f"cd{n}_A"], d[f"cd{n}_B"] = A, B
        spec = rc.circulant_decompose(A)
        d[f"cd{n}_cols"], d[f"cd{n}_mags"] = spec.columns, spec.magnitudes
        sel = rc.circulant_select(spec, k)
        d[f"cd{n}_sel"] = np.array(sel.selected, dtype=np.int64)
        d[f"cd{n}_mat"] = rc.circulant_materialize(sel)
        for order in (0, 1):
            M, rep = rc.circulant_first_order_multiply(A, B, k, order)
            d[f"cd{n}_M{order}"], d[f"cd{n}_rep{order}"] = M, rep_arr(rep)
        d[f"cd{n}_k"] = np.array(k)
    # complex input (root-of-unity diagonal, test_circulant.py:24-31 style)
    D = np.diag(np.exp(2j * np.pi * np.arange(6) / 6))
    d["cdz_A"] = D
    d["cdz_cols"] = rc.circulant_decompose(D).columns
    np.savez_compressed(os.path.join(OUT, "circulant.npz"), **d)


def svd_cases():
    d = {}
    rng = np.random.default_rng(300)
    for n, s, q, seed in [(16, 1, 0, 3), (32, 2, 1, 5), (64, 1, 0, 9), (64, 2, 2, 11)]:
        A = rng.standard_normal((n, n))
        B = rng.standard_normal((n, n))
        tag = f"svd{n}_{s}_{q}"
        d[tag + "_A"], d[tag + "_B"] = A, B
        d[tag + "_par"] = np.array([n, s, q, seed])
        for order in (0, 1):
            M, rep = rs.svd_first_order_multiply(A, B, s, order, seed=seed, power_iterations=q)
            d[tag + f"_M{order}"], d[tag + f"_rep{order}"] = M, rep_arr(rep)
        dec = rs.randomized_partial_svd(A, s, seed=seed, power_iterations=q)
        d[tag + "_U"], d[tag + "_S"], d[tag + "_V"] = dec.U, dec.sigma, dec.V
    # C1-style composition: oversampling p via components=k+p, truncate to k, order 0
    n, k, p, q, t = 64, 8, 4, 2, 1
    sig = 0.9 ** np.arange(n)
    A = apxmm.generate(apxmm.MatrixSpec("haar-spectrum", n, 2 * t, spectrum=sig))
    B = apxmm.generate(apxmm.MatrixSpec("haar-spectrum", n, 2 * t + 1, spectrum=sig))
    da = rs.randomized_partial_svd(A, 1, np.random.default_rng([t, 0]), power_iterations=q,
                                   components=k + p)
    db = rs.randomized_partial_svd(B, 1, np.random.default_rng([t, 1]), power_iterations=q,
                                   components=k + p)
    da = rs.TruncatedSVD(da.U[:, :k], da.sigma[:k], da.V[:, :k], da.source_frobenius_sq)
    db = rs.TruncatedSVD(db.U[:, :k], db.sigma[:k], db.V[:, :k], db.source_frobenius_sq)
    core = (da.V.T @ db.U) * db.sigma
    d["c1_A"], d["c1_B"] = A, B
    d["c1_par"] = np.array([n, k, p, q, t])
    d["c1_M"] = (da.U * da.sigma) @ (core @ db.V.T)
    d["c1_nd"] = np.array([rs.svd_residual_norm(da), rs.svd_residual_norm(db)])
    np.savez_compressed(os.path.join(OUT, "svd.npz"), **d)


def fsparse_cases():
    d = {}
    rng = np.random.default_rng(400)
    cases = [("sq16", (16, 16), (16, 16), 3), ("sq32", (32, 32), (32, 32), 5),
             ("rect", (12, 16), (16, 10), 4), ("full", (8, 8), (8, 8), 8),
             ("zero", (8, 8), (8, 8), 0)]
    for tag, sa, sb, k in cases:
        A = rng.standard_normal(sa)
        B = rng.standard_normal(sb)
        d[tag + "_A"], d[tag + "_B"], d[tag + "_k"] = A, B, np.array(k)
        for order in (0, 1):
            for mode in ("rows", "cols"):
                M, rep = rf.fft_sparse_first_order_multiply(A, B, k, order, sparsify_b=mode)
                d[f"{tag}_M{order}{mode}"] = M
                d[f"{tag}_rep{order}{mode}"] = rep_arr(rep)
    T = np.array([[1.0, -3.0, 3.0, 2.0], [0.0, 1.0, 1.0, -1.0]])
    d["tk_T"] = T
    for k in range(0, 6):
        d[f"tk_{k}"] = rf.topk_sparsify(T, k).to_dense()
    # fourier_row_decompose (fsparse.py:92-105): real, complex, n = 1, a rank-one row structure
    # (all weight in f_0: zero directions elsewhere), an odd length
    rf_rng = np.random.default_rng(401)
    frs = {"real": rf_rng.standard_normal((5, 8)),
           "cplx": rf_rng.standard_normal((7, 16)) + 1j * rf_rng.standard_normal((7, 16)),
           "n1": rf_rng.standard_normal((3, 1)),
           "const": np.outer(rf_rng.standard_normal(4), np.ones(6)),
           "odd": rf_rng.standard_normal((6, 97))}
    for tag, X in frs.items():
        spec = rf.fourier_row_decompose(X)
        d[f"frs_{tag}_A"], d[f"frs_{tag}_w"], d[f"frs_{tag}_d"] = X, spec.weights, spec.directions
    np.savez_compressed(os.path.join(OUT, "fsparse.npz"), **d)


def ref_cycle_decompose(A, k):
    lay = rcore.cycle_reorder(A, "left")
    norms = np.linalg.norm(lay, axis=0)
    J = rc.top_indices(norms, k)
    return J, lay, norms


def ref_cycle_product(A, B, ka, kb, order):
    """Compose the cycle product from reference primitives only."""
    n = A.shape[0]
    Ja, la, _ = ref_cycle_decompose(A, ka)
    Jb, lb, _ = ref_cycle_decompose(B, kb)
    keep_b = np.zeros_like(lb)
    keep_b[:, Jb] = lb[:, Jb]
    Bhat = rcore.cycle_reorder_inverse(keep_b, "left")
    X = Bhat if order == 0 else B
    M = np.zeros((n, n))
    for j in Ja:  # Lambda_j C^j X
        M += la[:, j][:, None] * rcore.apply_cycle_power(X, j, "left")
    if order == 1:
        resid = la.copy()
        resid[:, Ja] = 0.0
        dA = rcore.cycle_reorder_inverse(resid, "left")
        for j in Jb:  # dA Lambda_j C^j
            M += rcore.apply_cycle_power(dA * lb[:, j][None, :], j, "right")
    return M, Ja, Jb


def cycle_cases():
    sys.path.insert(0, os.path.dirname(os.path.dirname(OUT)))
    from oracle import gen_cycle_operand  # input generator only
    d = {}
    for n, ka, kb, ncyc in [(16, 3, 3, 3), (31, 4, 5, 4), (64, 8, 8, 8), (64, 6, 10, 12)]:
        A = gen_cycle_operand(n, ncyc, 2 * n)
        B = gen_cycle_operand(n, ncyc, 2 * n + 1)
        tag = f"cy{n}_{ka}_{kb}"
        d[tag + "_A"], d[tag + "_B"] = A, B
        for order in (0, 1):
            M, Ja, Jb = ref_cycle_product(A, B, ka, kb, order)
            d[tag + f"_M{order}"] = M
        d[tag + "_Ja"], d[tag + "_Jb"] = np.array(Ja), np.array(Jb)
    # mixed: A by reference rSVD (components=k), B by cycles
    n, ks, kc, seed = 64, 8, 6, 7
    A = apxmm.generate(apxmm.MatrixSpec("haar-spectrum", n, 14,
                                        spectrum=(np.arange(n) + 1.0) ** -1.5))
    B = gen_cycle_operand(n, kc, 15)
    da = rs.randomized_partial_svd(A, 1, np.random.default_rng([seed, 0]), components=ks)
    Jb, lb, _ = ref_cycle_decompose(B, kc)
    keep = np.zeros_like(lb)
    keep[:, Jb] = lb[:, Jb]
    Bhat = rcore.cycle_reorder_inverse(keep, "left")
    Ahat = rs.svd_reconstruct(da)
    d["mx_A"], d["mx_B"], d["mx_par"] = A, B, np.array([n, ks, kc, seed])
    d["mx_M0"] = Ahat @ Bhat
    d["mx_M1"] = Ahat @ B + (A - Ahat) @ Bhat
    d["mx_Jb"] = np.array(Jb)
    np.savez_compressed(os.path.join(OUT, "cycle.npz"), **d)


def errest_cases():
    from apxmm import errest as re_
    d = {}
    rng = np.random.default_rng(300)
    cases = [
        ("sq", rng.standard_normal((32, 32)), rng.standard_normal((32, 32)), 4, 7),
        ("rect", rng.standard_normal((17, 40)), rng.standard_normal((40, 23)), 5, 11),
        ("cplx", rng.standard_normal((12, 9)) + 1j * rng.standard_normal((12, 9)),
         rng.standard_normal((9, 14)) - 0.5j * rng.standard_normal((9, 14)), 3, 2),
        ("half", rng.standard_normal((10, 10)), rng.standard_normal((10, 10)) + 1j * rng.standard_normal((10, 10)),
         6, 5),
        ("zero", np.zeros((4, 4)), np.eye(4), 3, 0),
        ("wide", rng.standard_normal((3, 300)), rng.standard_normal((300, 2)), 64, 99),
    ]
    for name, A, B, k, seed in cases:
        d[f"sk_{name}_A"], d[f"sk_{name}_B"] = A, B
        d[f"sk_{name}_par"] = np.array([k, seed])
        d[f"sk_{name}_out"] = np.array(re_.sketch_norm_estimate(A, B, k, seed))
    d["sk_names"] = np.array([c[0] for c in cases])
    np.savez_compressed(os.path.join(OUT, "errest.npz"), **d)


def genmat_cases():
    """genmat.py:109-153 outputs for the value-exact kinds (the device generators reproduce them)."""
    from apxmm import genmat as rg

    d = {}
    for kind in ("toeplitz", "hankel", "block-toeplitz", "symmetric", "general", "circulant", "kappa"):
        for n in (1, 2, 5, 12, 36):
            d[f"{kind}_{n}"] = rg.generate(rg.MatrixSpec(kind, n, seed=3))
    d["block-toeplitz_12_b3"] = rg.generate(rg.MatrixSpec("block-toeplitz", 12, seed=4, block=3))
    np.savez_compressed(os.path.join(OUT, "genmat.npz"), **d)


if __name__ == "__main__":
    only = sys.argv[1:]
    for fn in (core_cases, circulant_cases, svd_cases, fsparse_cases, cycle_cases, errest_cases, genmat_cases):
        if not only or fn.__name__ in only:
            fn()
    for f in sorted(os.listdir(OUT)):
        if f.endswith(".npz"):
            print(f, os.path.getsize(os.path.join(OUT, f)))
