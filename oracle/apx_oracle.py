"""CPU oracle: a numpy restatement of the reference ``apxmm`` hot path (TEST INFRASTRUCTURE ONLY).

Each function names the reference lines (``/root/reference/pkg/src/apxmm/<file>:<line>``) whose
behaviour it restates. The code is written independently (explicit index arithmetic, plain loops
where the reference uses fancy indexing) so that it can serve as a checker; it follows the
reference's *evaluation order* wherever the result depends on it (ascending component order,
energy-difference residual norms, stable tie rule), because the GPU parity bar is measured
against the reference's approximation, not against exact AB.

Restated paths that the reference does not ship (``SURVEY.md`` §8(c)):
  * cycle-truncated product ``A = sum_j Lambda_j C^j`` (left layout, ``core.py:113,123-124``)
  * mixed product (rSVD for A x cycles for B, config C4)
  * rSVD oversampling (``components = k + p`` then truncate to k, config C1)
"""

from __future__ import annotations

import os
import math
import time

import numpy as np

__all__ = [
    "as_matrix", "unitary_dft", "cycle_reorder", "cycle_reorder_inverse", "apply_cycle_power",
    "frobenius", "relative_error", "top_indices", "component_count", "apriori_relative_error",
    "posterior_relative_error", "sketch_norm_estimate", "rsvd", "svd_first_order_multiply", "circulant_decompose",
    "circulant_materialize", "circulant_left_product", "circulant_right_product",
    "circulant_first_order_multiply", "topk_rows", "fourier_row_decompose", "fft_sparse_first_order_multiply",
    "cycle_product_rows",
    "cycle_norms", "cycle_decompose", "cycle_materialize", "cycle_first_order_multiply",
    "mixed_first_order_multiply", "gen_haar_spectrum", "gen_cycle_operand",
    "gen_circulant_operand", "gen_c5_operand", "Report",
]


# ----------------------------------------------------------------------------------------------
# core.py
# ----------------------------------------------------------------------------------------------

def as_matrix(a, allow_complex: bool = True) -> np.ndarray:
    """core.py:24-45 -- 2-D, non-empty, finite; cast to float64 / complex128."""
    m = np.asarray(a)
    if m.ndim != 2:
        raise ValueError(f"expected a 2-D matrix, got ndim={m.ndim}")
    if m.size == 0:
        raise ValueError("empty matrix")
    if np.iscomplexobj(m):
        if not allow_complex:
            raise ValueError("complex entries not allowed here")
        m = m.astype(np.complex128, copy=False)
        ok = np.isfinite(m.real).all() and np.isfinite(m.imag).all()
    else:
        m = m.astype(np.float64, copy=False)
        ok = np.isfinite(m).all()
    if not ok:
        raise ValueError("matrix entries must be finite (no NaN/Inf)")
    return m


def unitary_dft(x, direction: str = "forward", axis: int = -1) -> np.ndarray:
    """core.py:82-97 -- W (forward) or W* (inverse) along ``axis``, W(p,q)=e^{-2i pi pq/n}/sqrt(n)."""
    x = np.asarray(x)
    if x.ndim == 0 or x.shape[axis] < 1:
        raise ValueError("transform length must be >= 1")
    if direction == "forward":
        return np.fft.fft(x, axis=axis, norm="ortho")
    if direction == "inverse":
        return np.fft.ifft(x, axis=axis, norm="ortho")
    raise ValueError(f"unknown direction {direction!r}")


def _square(A) -> int:
    if A.shape[0] != A.shape[1]:
        raise ValueError(f"square matrix required, got {A.shape}")
    return A.shape[0]


def cycle_reorder(A, side: str) -> np.ndarray:
    """core.py:106-125.  right: out[i,j] = A[(i+j)%n, i];  left: out[i,j] = A[i, (i-j)%n]."""
    A = as_matrix(A)
    n = _square(A)
    i = np.arange(n)[:, None]
    j = np.arange(n)[None, :]
    if side == "right":
        return A[(i + j) % n, np.broadcast_to(i, (n, n))]
    if side == "left":
        return A[np.broadcast_to(i, (n, n)), (i - j) % n]
    raise ValueError(f"unknown side {side!r}")


def cycle_reorder_inverse(At, side: str) -> np.ndarray:
    """core.py:128-137 -- scatter the cycle columns back to their matrix positions."""
    At = as_matrix(At)
    n = _square(At)
    r = np.arange(n)[:, None]
    c = np.arange(n)[None, :]
    if side == "right":
        # A[r, c] sits in column j=(r-c)%n at row i=c of the right layout
        return At[np.broadcast_to(c, (n, n)), (r - c) % n]
    if side == "left":
        return At[np.broadcast_to(r, (n, n)), (r - c) % n]
    raise ValueError(f"unknown side {side!r}")


def apply_cycle_power(M, k: int, side: str) -> np.ndarray:
    """core.py:140-154 -- left: C^k M (rows rotate down by k); right: M C^k (cols rotate left)."""
    M = as_matrix(M)
    n = M.shape[0] if side == "left" else M.shape[1]
    if not 0 <= k < n:
        raise ValueError(f"k={k} out of range [0, {n})")
    if side == "left":
        return np.roll(M, k, axis=0)
    if side == "right":
        return np.roll(M, -k, axis=1)
    raise ValueError(f"unknown side {side!r}")


def frobenius(A, B=None):
    """core.py:64-79 -- ||A||_F, or <A,B>_F = sum(conj(A) * B)."""
    A = as_matrix(A)
    if B is None:
        return float(np.linalg.norm(A))
    B = as_matrix(B)
    if A.shape != B.shape:
        raise ValueError(f"shape mismatch: {A.shape} vs {B.shape}")
    v = np.vdot(A, B)
    if np.iscomplexobj(A) or np.iscomplexobj(B):
        return complex(v)
    return float(v.real)


def relative_error(M, C_ref) -> float:
    """core.py:157-166 -- ||C_ref - M||_F / ||C_ref||_F."""
    M = as_matrix(M)
    C_ref = as_matrix(C_ref)
    if M.shape != C_ref.shape:
        raise ValueError(f"shape mismatch: {M.shape} vs {C_ref.shape}")
    d = np.linalg.norm(C_ref)
    if d == 0.0:
        raise ValueError("zero-norm reference")
    return float(np.linalg.norm(C_ref - M) / d)


def top_indices(weights, k: int) -> list[int]:
    """circulant.py:63-70 -- k largest, ties toward the lower index, returned ascending.

    Restated as an explicit (value descending, index ascending) lexicographic order, which is
    what a stable argsort of -w produces.
    """
    w = np.asarray(weights)
    if not 0 <= k <= w.size:
        raise ValueError(f"k={k} out of range [0, {w.size}]")
    order = np.lexsort((np.arange(w.size), -w))
    return sorted(int(i) for i in order[:k])


# ----------------------------------------------------------------------------------------------
# errest.py (host scalars that end every multiply) and report.py
# ----------------------------------------------------------------------------------------------

def apriori_relative_error(normA, normB, ndA, ndB, n, case="mean-zero", c=None) -> float:
    """errest.py:108-124 with ErrorModel.product_constant errest.py:58-66."""
    if case == "mean-zero":
        cprod = 1.0 / math.sqrt(n)
    elif case == "unsigned":
        cprod = 0.75
    else:
        cprod = float(c)
    return (ndA * ndB / math.sqrt(n)) / (cprod * normA * normB)


def posterior_relative_error(ndA, ndB, normM, n) -> float:
    """errest.py:127-136."""
    return ndA * ndB / (math.sqrt(n) * normM)


def sketch_norm_estimate(A, B, k: int, seed) -> float:
    """errest.py:139-154 -- ||A (B G)||_F^2 / k, G = default_rng(seed).standard_normal((cols(B), k))."""
    A = as_matrix(A)
    B = as_matrix(B)
    if A.shape[1] != B.shape[0]:
        raise ValueError("dimension mismatch")
    if k < 1:
        raise ValueError("k must be >= 1")
    G = np.random.default_rng(seed).standard_normal((B.shape[1], k))
    T = A @ (B @ G)
    return float(np.sum(np.abs(T) ** 2) / k)


class Report(dict):
    """Fields of ApproxReport (report.py:8-36) as a plain dict."""


def _report(method, order, k, normA, normB, ndA, ndB, M, n, wall):
    apri = (apriori_relative_error(normA, normB, ndA, ndB, n)
            if normA > 0 and normB > 0 else None)
    nM = float(np.linalg.norm(M))
    post = posterior_relative_error(ndA, ndB, nM, n) if nM > 0 else None
    return Report(method=method, order=order, k=k, norm_da=ndA, norm_db=ndB,
                  apriori_estimate=apri, posterior_estimate=post, measured_error=None,
                  wall_time=wall, norm_m=nM)


# ----------------------------------------------------------------------------------------------
# svd.py
# ----------------------------------------------------------------------------------------------

def component_count(n: int, s: int) -> int:
    """svd.py:72-80 -- k = min(s*floor(log2 n)+1, n); n=1 -> 1."""
    if n < 1:
        raise ValueError("n must be >= 1")
    if s < 1:
        raise ValueError("s must be >= 1")
    if n == 1:
        return 1
    return min(s * int(math.floor(math.log2(n))) + 1, n)


def rsvd(A, k: int, rng, power_iterations: int = 0):
    """svd.py:83-119 (Alg. 2.1) with the sketch width given directly (``components=``).

    Returns (U, sigma, V, ||A||_F^2). The sketch draws ``rng.standard_normal((n, k))`` exactly
    like svd.py:105-106, so a shared seed gives the identical Omega.
    """
    A = as_matrix(A, allow_complex=False)
    m, n = A.shape
    k = min(k, m, n)
    if not isinstance(rng, np.random.Generator):
        rng = np.random.default_rng(rng)
    omega = rng.standard_normal((n, k))
    Q = np.linalg.qr(A @ omega, mode="reduced")[0]
    for _ in range(power_iterations):
        Q = np.linalg.qr(A.T @ Q, mode="reduced")[0]
        Q = np.linalg.qr(A @ Q, mode="reduced")[0]
    Ub, s, Vt = np.linalg.svd(Q.T @ A, full_matrices=False)
    return Q @ Ub, s, Vt.T, float(np.linalg.norm(A) ** 2)


def _svd_resid(sigma, fro2) -> float:
    """svd.py:122-130 -- energy difference, clamped at 0."""
    return math.sqrt(max(0.0, fro2 - float(np.sum(sigma ** 2))))


def _truncate(U, s, V, k):
    return U[:, :k], s[:k], V[:, :k]


def svd_first_order_multiply(A, B, s: int | None, order: int, seed, power_iterations: int = 0,
                             components: int | None = None, oversampling: int = 0):
    """svd.py:138-200.  ``components``/``oversampling`` restate config C1 (k=32, p=8): sketch
    k+p columns through the reference algorithm, then keep the leading k triplets.
    Seeds: default_rng([seed,0]) for A, default_rng([seed,1]) for B (svd.py:161-162)."""
    A = as_matrix(A, allow_complex=False)
    B = as_matrix(B, allow_complex=False)
    if A.shape[1] != B.shape[0]:
        raise ValueError(f"dimension mismatch: {A.shape} x {B.shape}")
    if order not in (0, 1):
        raise ValueError("order must be 0 or 1")
    t0 = time.perf_counter()
    if components is None:
        ka = min(component_count(A.shape[1], s), A.shape[0])
        kb = min(component_count(B.shape[1], s), B.shape[0])
    else:
        ka = kb = components
    ra = np.random.default_rng([seed, 0])
    rb = np.random.default_rng([seed, 1])
    Ua, sa, Va, fa = rsvd(A, ka + oversampling, ra, power_iterations)
    Ub, sb, Vb, fb = rsvd(B, kb + oversampling, rb, power_iterations)
    if oversampling:
        Ua, sa, Va = _truncate(Ua, sa, Va, ka)
        Ub, sb, Vb = _truncate(Ub, sb, Vb, kb)
    ndA, ndB = _svd_resid(sa, fa), _svd_resid(sb, fb)
    Uas = Ua * sa
    if order == 0:
        core = (Va.T @ Ub) * sb
        M = Uas @ (core @ Vb.T)
    else:
        term1 = Uas @ (Va.T @ B)
        dA = A - (Ua * sa) @ Va.T
        M = term1 + ((dA @ Ub) * sb) @ Vb.T
    wall = time.perf_counter() - t0
    rep = _report("svd", order, sa.size, math.sqrt(fa), math.sqrt(fb), ndA, ndB, M,
                  A.shape[1], wall)
    return M, rep


# ----------------------------------------------------------------------------------------------
# circulant.py
# ----------------------------------------------------------------------------------------------

def circulant_decompose(A):
    """circulant.py:73-91 -- S = W.cycle_reorder(A,'right')/sqrt(n) (axis 0); mags = row norms."""
    A = as_matrix(A)
    n = _square(A)
    S = unitary_dft(cycle_reorder(A, "right"), "forward", axis=0) / math.sqrt(n)
    return S, np.linalg.norm(S, axis=1)


def circulant_materialize(S, selected) -> np.ndarray:
    """circulant.py:116-127 -- sum_{t in sel} S[t][(r-c)%n] * omega^{t c}, ascending t."""
    n = S.shape[0]
    out = np.zeros((n, n), dtype=np.complex128)
    r = np.arange(n)[:, None]
    c = np.arange(n)[None, :]
    diff = (r - c) % n
    for t in selected:
        phase = np.exp(2j * np.pi * ((t * np.arange(n)) % n) / n)
        out += S[t][diff] * phase[None, :]
    return out


def circulant_left_product(S, selected, FB) -> np.ndarray:
    """circulant.py:136-147 -- W* sum_t diag(fft(S[t])) C^t FB, ascending t."""
    acc = np.zeros(FB.shape, dtype=np.complex128)
    for t in selected:
        L = np.fft.fft(S[t])
        acc += L[:, None] * np.roll(FB, t, axis=0)
    return unitary_dft(acc, "inverse", axis=0)


def circulant_right_product(S, selected, G) -> np.ndarray:
    """circulant.py:150-161 -- G sum_t R_t D^t evaluated on G^H in the Fourier domain."""
    X = unitary_dft(np.conj(G).T, "forward", axis=0)
    acc = np.zeros(X.shape, dtype=np.complex128)
    for t in selected:
        L = np.fft.fft(S[t])
        acc += np.roll(np.conj(L)[:, None] * X, -t, axis=0)
    return np.conj(unitary_dft(acc, "inverse", axis=0)).T


def circulant_first_order_multiply(A, B, k: int, order: int, force_sel_a=None, force_sel_b=None):
    """circulant.py:164-218.  ``force_sel_*`` implement the near-tie protocol:
    re-run with the GPU's index list, as the reference tests do (test_circulant.py:108-110)."""
    A = as_matrix(A)
    B = as_matrix(B)
    n = A.shape[0]
    if A.shape[1] != n or B.shape != (n, n):
        raise ValueError(f"two square n x n matrices required, got {A.shape} x {B.shape}")
    if not 0 <= k <= n:
        raise ValueError(f"k={k} out of range [0, {n}]")
    if order not in (0, 1):
        raise ValueError("order must be 0 or 1")
    t0 = time.perf_counter()
    Sa, ma = circulant_decompose(A)
    Sb, mb = circulant_decompose(B)
    sel_a = list(force_sel_a) if force_sel_a is not None else top_indices(ma, k)
    sel_b = list(force_sel_b) if force_sel_b is not None else top_indices(mb, k)
    nA, nB = float(np.linalg.norm(A)), float(np.linalg.norm(B))
    ndA = math.sqrt(max(0.0, nA ** 2 - n * sum(float(ma[t]) ** 2 for t in sel_a)))
    ndB = math.sqrt(max(0.0, nB ** 2 - n * sum(float(mb[t]) ** 2 for t in sel_b)))
    M = circulant_left_product(Sa, sel_a, unitary_dft(B, "forward", axis=0))
    if order == 1:
        dA = A - circulant_materialize(Sa, sel_a)
        M = M + circulant_right_product(Sb, sel_b, dA)
    wall = time.perf_counter() - t0
    rep = _report("cd", order, k, nA, nB, ndA, ndB, M, n, wall)
    rep["selected_a"], rep["selected_b"] = sel_a, sel_b
    rep["magnitudes_a"], rep["magnitudes_b"] = ma, mb
    return M, rep


# ----------------------------------------------------------------------------------------------
# fsparse.py (secondary path)
# ----------------------------------------------------------------------------------------------

def topk_rows(M, k, force=None):
    """fsparse.py:108-139 -- per-row k largest |.|, ties to the lower column; dense masked copy.
    ``force`` (per-row column lists) replaces the selection (near-tie protocol).

    Returns (dense matrix holding only the kept entries, list of ascending column lists)."""
    M = as_matrix(M)
    rows, cols = M.shape
    if force is not None:
        out = np.zeros((rows, cols), dtype=np.complex128)
        for i, keep in enumerate(force):
            out[i, list(keep)] = M[i, list(keep)]
        return out, [sorted(int(j) for j in keep) for keep in force]
    if np.isscalar(k):
        if k < 0:
            raise ValueError("k must be >= 0")
        budgets = [min(int(k), cols)] * rows
    else:
        budgets = [min(int(v), cols) for v in k]
        if len(budgets) != rows:
            raise ValueError("need one budget per row")
    out = np.zeros((rows, cols), dtype=np.complex128)
    lists = []
    for i in range(rows):
        if budgets[i] == 0:
            lists.append([])
            continue
        mag = np.abs(M[i])
        order = np.lexsort((np.arange(cols), -mag))[:budgets[i]]
        keep = sorted(int(j) for j in order)
        out[i, keep] = M[i, keep]
        lists.append(keep)
    return out, lists


def fourier_row_decompose(A):
    """fsparse.py:92-105 -- F = W(rows)/sqrt(n); weights sqrt(n)||f_k||, unit directions, zero
    columns where the weight vanishes. Returns (weights, directions)."""
    A = as_matrix(A)
    n = A.shape[1]
    F = unitary_dft(A, "forward", axis=1) / math.sqrt(n)
    col = np.linalg.norm(F, axis=0)
    directions = np.zeros_like(F)
    nz = col > 0
    directions[:, nz] = F[:, nz] / col[nz]
    return math.sqrt(n) * col, directions


def fft_sparse_first_order_multiply(A, B, k: int, order: int, sparsify_b: str = "rows", force_a=None,
                                    force_b=None):
    """fsparse.py:168-240 -- At = A W*, Bt = W B, per-row top-k of both, first-order product."""
    A = as_matrix(A)
    B = as_matrix(B)
    n = A.shape[1]
    if B.shape[0] != n:
        raise ValueError(f"dimension mismatch: {A.shape} x {B.shape}")
    if k < 0:
        raise ValueError(f"k={k} must be >= 0")
    if order not in (0, 1):
        raise ValueError("order must be 0 or 1")
    if sparsify_b not in ("rows", "cols"):
        raise ValueError(f"unknown sparsify_b {sparsify_b!r}")
    t0 = time.perf_counter()
    At = unitary_dft(A, "inverse", axis=1)
    Bt = unitary_dft(B, "forward", axis=0)
    SA, la = topk_rows(At, k, force_a)
    if sparsify_b == "rows":
        SB, lb = topk_rows(Bt, k, force_b)
    else:
        SBt, lb = topk_rows(Bt.T, k, force_b)
        SB = SBt.T
    dAt = At - SA
    ndA, ndB = float(np.linalg.norm(dAt)), float(np.linalg.norm(Bt - SB))
    if order == 0:
        M = SA @ SB
    else:
        M = SA @ Bt + dAt @ SB
    wall = time.perf_counter() - t0
    rep = _report("sfft", order, k, float(np.linalg.norm(A)), float(np.linalg.norm(B)),
                  ndA, ndB, M, n, wall)
    rep["selected_a"], rep["selected_b"] = la, lb
    rep["At"], rep["Bt"] = At, Bt
    return M, rep


# ----------------------------------------------------------------------------------------------
# cycle-truncated product (restated; no reference function -- PAPER.md:46-58, core.py:106-154)
# ----------------------------------------------------------------------------------------------

def cycle_norms(A) -> np.ndarray:
    """Column 2-norms of cycle_reorder(A, 'left') (core.py:123-124): ||lambda_j||_2 for each j."""
    return np.linalg.norm(cycle_reorder(A, "left"), axis=0)


def _cycle_norms_blocked(A, block: int = 256) -> np.ndarray:
    """Column 2-norms of cycle_reorder(A, 'left') without the n x n index arrays: the layout is
    gathered one row block at a time and the squares are accumulated row by row in ascending row
    order -- the order of numpy's add.reduce along axis 0 in np.linalg.norm(lay, axis=0), so the
    result is bitwise the full-layout one (checked in tests/test_oracle_golden.py)."""
    n = A.shape[0]
    acc = np.zeros((1, n))
    j = np.arange(n)[None, :]
    for r0 in range(0, n, block):
        i = np.arange(r0, min(n, r0 + block))[:, None]
        lay = A[i, (i - j) % n]
        acc = np.add.reduce(np.concatenate([acc, lay * lay], axis=0), axis=0, keepdims=True)
    return np.sqrt(acc[0])


def cycle_decompose(A, k: int, force_sel=None):
    """Dominant-cycle split A = sum_{j in J} Lambda_j C^j + dA.

    Selection follows top_indices (circulant.py:63-70) on the cycle norms; returns
    (J ascending, lambdas k x n with lambdas[t][i] = A[i,(i-J[t])%n], norms, ||A||, ||dA||)."""
    A = as_matrix(A, allow_complex=False)
    n = _square(A)
    if not 0 <= k <= n:
        raise ValueError(f"k={k} out of range [0, {n}]")
    norms = _cycle_norms_blocked(A)
    J = list(force_sel) if force_sel is not None else top_indices(norms, k)
    i = np.arange(n)
    lam = np.ascontiguousarray(np.array([A[i, (i - j) % n] for j in J]).reshape(len(J), n))
    nA = float(np.linalg.norm(A))
    nd = math.sqrt(max(0.0, nA ** 2 - sum(float(norms[j]) ** 2 for j in J)))
    return J, lam, norms, nA, nd


def cycle_materialize(J, lam, n) -> np.ndarray:
    """sum_t Lambda_t C^{J[t]} as a dense matrix (Lambda_t C^j has lam[t][i] at (i,(i-j)%n))."""
    lay = np.zeros((n, n))
    for t, j in enumerate(J):
        lay[:, j] = lam[t]
    return cycle_reorder_inverse(lay, "left")


def _cycle_residual(A, J) -> np.ndarray:
    """dA = A with the kept cycles zeroed (cycles partition the entries)."""
    lay = cycle_reorder(A, "left")
    lay[:, J] = 0.0
    return cycle_reorder_inverse(lay, "left")


def _cycle_left_apply(J, lam, X, rows=None) -> np.ndarray:
    """(sum_t Lambda_t C^{J[t]}) X = sum_t lam_t o apply_cycle_power(X, J[t], 'left'), ascending t.
    ``rows`` restricts the output to a row subset (the bounded CPU sample)."""
    n = X.shape[0]
    r = np.arange(n) if rows is None else np.asarray(rows)
    out = np.zeros((r.size, X.shape[1]), dtype=np.result_type(X, lam))
    for t, j in enumerate(J):
        out += lam[t][r][:, None] * X[(r - j) % n]
    return out


def _cycle_right_apply(X, J, lam) -> np.ndarray:
    """X (sum_t Lambda_t C^{J[t]}) = sum_t apply_cycle_power(X o lam_t, J[t], 'right'), ascending t.
    The roll by -j is written as two slice adds (out[:, c] += (X o lam_t)[:, (c + j) % n]): the same
    values in the same order as np.roll, without its temporary."""
    out = np.zeros(X.shape, dtype=np.result_type(X, lam))
    tmp = np.empty(X.shape, dtype=out.dtype)
    n = X.shape[1]
    for t, j in enumerate(J):
        j = int(j) % n
        np.multiply(X, lam[t][None, :], out=tmp)
        out[:, : n - j] += tmp[:, j:]
        if j:
            out[:, n - j:] += tmp[:, :j]
    return out


def cycle_product_rows(rows, A_rows, JA, B_shifted_rows, JB, lamB):
    """Rows R of the order-1 cycle product from row data only (config C5: n too large for the
    full oracle): M[R,:] = sum_t lamA_t[R] B[(R-JA_t)%n, :] + dA[R,:] . Bhat.

    A_rows: A[R, :]; B_shifted_rows[t]: B[(R - JA[t]) % n, :]; lamB: kb x n left-layout lambdas of
    B (core.py:123-124).  term1 follows _cycle_left_apply, term2 _cycle_right_apply on dA[R, :],
    dA = A with the kept cycles zeroed (_cycle_residual)."""
    R = np.asarray(rows)
    A_rows = np.asarray(A_rows, dtype=np.float64)
    n = A_rows.shape[1]
    ri = np.arange(R.size)
    term1 = np.zeros(A_rows.shape)
    dA = A_rows.copy()
    for t, j in enumerate(JA):
        cols = (R - j) % n
        term1 += A_rows[ri, cols][:, None] * np.asarray(B_shifted_rows[t], dtype=np.float64)
        dA[ri, cols] = 0.0
    return term1 + _cycle_right_apply(dA, JB, np.asarray(lamB, dtype=np.float64))


def cycle_first_order_multiply(A, B, k: int, order: int, kb: int | None = None,
                               force_sel_a=None, force_sel_b=None):
    """Cycle-truncated product (config C2).  order 0: Ahat.Bhat (PAPER.md:126-133 zeroth order,
    the svd convention svd.py:169-172); order 1: Ahat.B + dA.Bhat (svd.py:174-177 structure)."""
    A = as_matrix(A, allow_complex=False)
    B = as_matrix(B, allow_complex=False)
    n = A.shape[0]
    if A.shape[1] != n or B.shape != (n, n):
        raise ValueError(f"two square n x n matrices required, got {A.shape} x {B.shape}")
    if order not in (0, 1):
        raise ValueError("order must be 0 or 1")
    kb = k if kb is None else kb
    t0 = time.perf_counter()
    Ja, la, na_, nA, ndA = cycle_decompose(A, k, force_sel_a)
    Jb, lb, nb_, nB, ndB = cycle_decompose(B, kb, force_sel_b)
    if order == 0:
        M = _cycle_left_apply(Ja, la, cycle_materialize(Jb, lb, n))
    else:
        M = _cycle_left_apply(Ja, la, B) + _cycle_right_apply(_cycle_residual(A, Ja), Jb, lb)
    wall = time.perf_counter() - t0
    rep = _report("cycle", order, k, nA, nB, ndA, ndB, M, n, wall)
    rep["selected_a"], rep["selected_b"] = Ja, Jb
    rep["norms_a"], rep["norms_b"] = na_, nb_
    return M, rep


def mixed_first_order_multiply(A, B, k_svd: int, k_cyc: int, order: int, seed,
                               power_iterations: int = 0, force_sel_b=None, rows=None, block: int = 64,
                               threads: int | None = None):
    """Mixed product (config C4): A by rSVD (svd.py:83-119, stream default_rng([seed,0])),
    B by its k_cyc dominant cycles.  order 1: Ahat.B + dA.Bhat (reference order);
    order 0: Ahat.Bhat.  ``rows`` evaluates only that row subset of M (bounded CPU sample)."""
    A = as_matrix(A, allow_complex=False)
    B = as_matrix(B, allow_complex=False)
    n = A.shape[0]
    if A.shape[1] != n or B.shape != (n, n):
        raise ValueError(f"two square n x n matrices required, got {A.shape} x {B.shape}")
    if order not in (0, 1):
        raise ValueError("order must be 0 or 1")
    t0 = time.perf_counter()
    U, s, V, fa = rsvd(A, k_svd, np.random.default_rng([seed, 0]), power_iterations)
    Jb, lb, nb_, nB, ndB = cycle_decompose(B, k_cyc, force_sel_b)
    t_dec = time.perf_counter() - t0
    r = np.arange(n) if rows is None else np.asarray(rows)
    Us = U[r] * s
    if order == 0:
        M = Us @ _cycle_right_apply(V.T, Jb, lb)
    else:
        # dense parts with the (multithreaded) BLAS, then the cycle term dA . Bhat over row blocks:
        # the blocks are independent (the same values whatever the thread count) and numpy
        # releases the GIL in their elementwise passes, so the host's cores share them
        M = Us @ (V.T @ B)
        dA = A[r] - Us @ V.T

        def rows_block(b0):
            M[b0:b0 + block] += _cycle_right_apply(dA[b0:b0 + block], Jb, lb)

        starts = list(range(0, r.size, block))
        nthr = max(1, min(len(starts), threads or os.cpu_count() or 1))
        if nthr == 1:
            for b0 in starts:
                rows_block(b0)
        else:
            from concurrent.futures import ThreadPoolExecutor
            with ThreadPoolExecutor(nthr) as ex:
                list(ex.map(rows_block, starts))
    wall = time.perf_counter() - t0
    rep = _report("mixed", order, s.size, math.sqrt(fa), nB, _svd_resid(s, fa), ndB, M, n, wall)
    rep["selected_b"], rep["norms_b"] = Jb, nb_
    rep["t_decompose"] = t_dec
    return M, rep


# ----------------------------------------------------------------------------------------------
# seeded synthetic operands for BASELINE.json configs; host-side numpy
# ----------------------------------------------------------------------------------------------

def _haar(rng, n):
    """genmat.py:94-99 -- sign-corrected QR of a Gaussian matrix."""
    Q, R = np.linalg.qr(rng.standard_normal((n, n)), mode="reduced")
    d = np.sign(np.diag(R))
    d[d == 0] = 1.0
    return Q * d[None, :]


def gen_haar_spectrum(n: int, sigma, seed: int) -> np.ndarray:
    """genmat.py:102-106,151-152 ('haar-spectrum', kind code 11): (Q1 diag(s)) Q2^T."""
    rng = np.random.default_rng([seed, 11, n])
    s = np.asarray(sigma, dtype=float)
    Q1 = _haar(rng, n)
    Q2 = _haar(rng, n)
    return (Q1 * s[None, :]) @ Q2.T


def gen_cycle_operand(n: int, ncyc: int, seed: int, noise: float = 1e-3) -> np.ndarray:
    """C2/C4-B: N(0, noise^2) residue plus ``ncyc`` dominant cycles with N(0,1) diagonals at
    distinct shifts drawn without replacement; stream default_rng([seed, 101, n])."""
    rng = np.random.default_rng([seed, 101, n])
    A = noise * rng.standard_normal((n, n))
    J = rng.choice(n, size=ncyc, replace=False)
    i = np.arange(n)
    for j in J:
        A[i, (i - j) % n] += rng.standard_normal(n)
    return A


def _smooth_circulant_column(rng, n):
    """c with N(0,1) spectrum scaled by 1/(1+f)^2, f = min(q, n-q); Hermitian -> real."""
    f = np.arange(n // 2 + 1)
    spec = np.fft.rfft(rng.standard_normal(n)) / (1.0 + f) ** 2
    return np.fft.irfft(spec, n)


def gen_circulant_operand(n: int, r: int, seed: int, noise: float = 1e-3) -> np.ndarray:
    """C3: sum_{i<r} diag(d_i) Circ(c_i) + N(0, noise^2), d_i ~ U(0.5,1.5), Circ[a,b]=c[(a-b)%n]
    (scipy.linalg.circulant convention, genmat.py:135-136); stream default_rng([seed, 102, n])."""
    rng = np.random.default_rng([seed, 102, n])
    A = noise * rng.standard_normal((n, n))
    idx = (np.arange(n)[:, None] - np.arange(n)[None, :]) % n
    for _ in range(r):
        d = rng.uniform(0.5, 1.5, n)
        c = _smooth_circulant_column(rng, n)
        A += d[:, None] * c[idx]
    return A


def gen_c5_operand(n: int, ncyc: int, r: int, seed: int, noise: float = 1e-3) -> np.ndarray:
    """C5 (small-n host version): cycles + circulant terms + noise; stream ([seed, 103, n])."""
    rng = np.random.default_rng([seed, 103, n])
    A = noise * rng.standard_normal((n, n))
    i = np.arange(n)
    for j in rng.choice(n, size=ncyc, replace=False):
        A[i, (i - j) % n] += rng.standard_normal(n)
    idx = (i[:, None] - i[None, :]) % n
    for _ in range(r):
        d = rng.uniform(0.5, 1.5, n)
        A += d[:, None] * _smooth_circulant_column(rng, n)[idx]
    return A
