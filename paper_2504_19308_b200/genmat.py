"""Device generators for the reference's matrix families and the BASELINE configs' synthetic
operands (reference genmat.py:109-153).

The O(n^2) materialisation runs on the device; the random draws follow one of two contracts:

* **exact** (the reference's stream): kinds whose randomness is an O(n) vector or a plain
  uniform matrix (toeplitz, hankel, block-toeplitz, circulant, symmetric, general) draw it with
  numpy's ``default_rng([seed, kind code, n])`` exactly as genmat.py:90-91 does, so the device
  matrix is bit-identical to ``apxmm.genmat.generate`` (pinned by tests/golden genmat vectors);
  ``kappa`` is deterministic and exact too.
* **distribution** (device Philox): the Haar-based kinds (type1, type2, type3, haar-spectrum) need
  an n x n QR of a Gaussian matrix, which the reference does with LAPACK on the host (71 s at
  n = 8192). Here the Gaussian comes from torch's Philox generator keyed by the seed and the QR
  from the device solver, with the same sign correction (genmat.py:94-99): the same distribution,
  not the same values.

The config operands (``cycle_operand``, ``circulant_operand``, ``c5_operand``, ``c4_operands``)
realise SURVEY.md §8(d)'s synthetic inputs on the device with Philox streams keyed per operand.
"""

from __future__ import annotations

import math

import numpy as np
import torch

__all__ = [
    "KIND_CODE", "EXACT_KINDS", "generate", "haar_orthogonal", "haar_spectrum", "cycle_operand",
    "smooth_circulant_column", "circulant_operand", "c5_operand", "c4_operands",
]

# genmat.py:31-43 (frozen stream identifiers)
KIND_CODE = {"toeplitz": 1, "hankel": 2, "block-toeplitz": 3, "symmetric": 4, "general": 5, "circulant": 6,
             "kappa": 7, "type1": 8, "type2": 9, "type3": 10, "haar-spectrum": 11}
EXACT_KINDS = ("toeplitz", "hankel", "block-toeplitz", "symmetric", "general", "circulant", "kappa")


def _default_block(n: int) -> int:
    """genmat.py:48-51 -- divisor of n closest to sqrt(n), ties toward the smaller divisor."""
    divisors = [d for d in range(1, n + 1) if n % d == 0]
    return min(divisors, key=lambda d: (abs(d - math.isqrt(n)), d))


def _philox(seed, device) -> torch.Generator:
    g = torch.Generator(device=device)
    g.manual_seed(int(np.random.SeedSequence(seed).generate_state(1, np.uint64)[0] & ((1 << 63) - 1)))
    return g


def haar_orthogonal(n: int, g: torch.Generator, device, dtype=torch.float64) -> torch.Tensor:
    """genmat.py:94-99 on the device: Q of QR(G), G ~ N(0,1) n x n, columns sign-corrected by
    sign(diag R) (0 -> +1)."""
    G = torch.randn(n, n, generator=g, device=device, dtype=torch.float64)
    Q, R = torch.linalg.qr(G)
    d = torch.sign(torch.diagonal(R))
    d[d == 0] = 1.0
    return (Q * d).to(dtype)


def haar_spectrum(n: int, sigma, seed, device="cuda", dtype=torch.float64, g: torch.Generator | None = None):
    """genmat.py:102-106: (Q1 diag(sigma)) Q2^T with Q1 then Q2 from one stream."""
    g = g if g is not None else _philox([seed, KIND_CODE["haar-spectrum"], n], device)
    s = torch.as_tensor(np.asarray(sigma, dtype=np.float64), device=device)
    Q1 = haar_orthogonal(n, g, device)
    Q2 = haar_orthogonal(n, g, device)
    A = (Q1 * s) @ Q2.T
    del Q1, Q2
    return A.to(dtype).contiguous()


def _toeplitz_from_d(d: torch.Tensor, n: int) -> torch.Tensor:
    """scipy.linalg.toeplitz(c=d[:n], r=[d0, d[n:]]): T[i, j] = f[n-1+i-j] with f[n-1+q] = d[q]
    (q >= 0) and f[n-1-m] = d[n-1+m] (m >= 1)."""
    f = torch.cat([d[n:].flip(0), d[:n]])
    return f.as_strided((n, n), (1, 1)).flip(1).contiguous()


def generate(kind: str, n: int, seed: int = 0, block: int | None = None, spectrum=None, device="cuda",
             dtype=torch.float64) -> torch.Tensor:
    """Device counterpart of ``apxmm.genmat.generate(MatrixSpec(kind, n, seed, block, spectrum))``
    (genmat.py:109-153); see the module docstring for which kinds are value-exact."""
    if kind not in KIND_CODE:
        raise ValueError(f"unknown kind {kind!r}; expected one of {tuple(KIND_CODE)}")
    if n < 1:
        raise ValueError("n must be >= 1")
    if kind == "block-toeplitz":
        block = _default_block(n) if block is None else block
        if block < 1 or n % block != 0:
            raise ValueError(f"block {block} must divide n={n}")
    elif block is not None:
        raise ValueError(f"kind {kind!r} takes no block size")
    if kind == "haar-spectrum":
        if spectrum is None:
            raise ValueError("haar-spectrum needs a spectrum vector")
        s = np.asarray(spectrum, dtype=float)
        if s.ndim != 1 or s.size != n:
            raise ValueError("spectrum must be a length-n vector")
        if np.any(s < 0) or not np.all(np.isfinite(s)):
            raise ValueError("spectrum values must be finite and >= 0")
    elif spectrum is not None:
        raise ValueError(f"kind {kind!r} takes no spectrum")
    rng = np.random.default_rng([seed, KIND_CODE[kind], n])  # genmat.py:90-91

    def dev(x):
        return torch.from_numpy(np.ascontiguousarray(x)).to(device)

    if kind == "toeplitz":
        out = _toeplitz_from_d(dev(rng.uniform(0.0, 1.0, 2 * n - 1)), n)
    elif kind == "hankel":
        d = dev(rng.uniform(0.0, 1.0, 2 * n - 1))
        out = d.as_strided((n, n), (1, 1)).contiguous()  # H[i, j] = d[i + j]
    elif kind == "block-toeplitz":
        nb = n // block
        blocks = dev(rng.uniform(0.0, 1.0, (2 * nb - 1, block, block)))
        bi = torch.arange(nb, device=device)
        idx = bi[:, None] - bi[None, :] + nb - 1  # block (i, j) = blocks[i - j + nb - 1]
        out = blocks[idx].permute(0, 2, 1, 3).reshape(n, n).contiguous()
    elif kind == "symmetric":
        G = dev(rng.uniform(0.0, 1.0, (n, n)))
        out = (G + G.T) / 2.0
    elif kind == "general":
        out = dev(rng.uniform(0.0, 1.0, (n, n)))
    elif kind == "circulant":
        c = dev(rng.uniform(0.0, 1.0, n))
        i = torch.arange(n, device=device)
        out = c[(i[:, None] - i[None, :]) % n]
    elif kind == "kappa":
        i = torch.arange(n, device=device, dtype=torch.float64)
        out = torch.exp(-0.5 * (i[:, None] - i[None, :]).abs()) * torch.sin(torch.minimum(i[:, None], i[None, :]) + 1.0)
    else:
        g = _philox([seed, KIND_CODE[kind], n], device)
        if kind == "type1":
            out = haar_spectrum(n, np.exp(-np.arange(n) / n), seed, device, g=g)
        elif kind == "type3":
            out = haar_spectrum(n, (n - np.arange(n)) / n, seed, device, g=g)
        elif kind == "haar-spectrum":
            out = haar_spectrum(n, spectrum, seed, device, g=g)
        else:  # type2: type1 + (0.5 ||T|| / ||U||) U, U uniform from the type2 stream
            T = generate("type1", n, seed, device=device)
            U = torch.rand(n, n, generator=g, device=device, dtype=torch.float64)
            out = T + (0.5 * torch.linalg.norm(T) / torch.linalg.norm(U)) * U
    return out.to(dtype).contiguous()


# ---- config operands -------------------------------------------------------

def cycle_operand(n: int, ncyc: int, seed: int, device="cuda", dtype=torch.float64, noise: float = 1e-3,
                  g: torch.Generator | None = None):
    """C2 / C4-B: N(0, noise^2) residue plus `ncyc` cycles with N(0,1) diagonals at distinct shifts
    (left layout core.py:123-124: cycle j at A[i, (i - j) % n]). Returns (A, shifts ascending)."""
    g = g if g is not None else _philox([seed, 101, n], device)
    A = noise * torch.randn(n, n, generator=g, device=device, dtype=dtype)
    J = torch.randperm(n, generator=g, device=device)[:ncyc]
    i = torch.arange(n, device=device)
    for j in J.tolist():
        A[i, (i - j) % n] += torch.randn(n, generator=g, device=device, dtype=dtype)
    return A, sorted(J.tolist())


def smooth_circulant_column(n: int, g: torch.Generator, device) -> torch.Tensor:
    """c with an N(0,1) spectrum scaled by 1/(1+f)^2, f = min(q, n-q); Hermitian, so c is real."""
    f = torch.arange(n // 2 + 1, device=device, dtype=torch.float64)
    spec = torch.fft.rfft(torch.randn(n, generator=g, device=device, dtype=torch.float64)) / (1.0 + f) ** 2
    return torch.fft.irfft(spec, n)


def _add_diag_circulant(A: torch.Tensor, d: torch.Tensor, c: torch.Tensor, chunk: int = 2048):
    """A += diag(d) Circ(c), Circ(c)[i, k] = c[(i - k) % n] (scipy.linalg.circulant), in row
    chunks (a row-flipped Hankel view of the wrapped column keeps every index in int32 range)."""
    n = A.shape[0]
    dd, cc = d.to(A.dtype), c.to(A.dtype)
    for s in range(0, n, chunk):
        cs = min(chunk, n - s)
        q = torch.arange(cs + n - 1, device=A.device)
        y = cc[(s + cs - 1 - q) % n].contiguous()
        A[s:s + cs].addcmul_(dd[s:s + cs, None], y.as_strided((cs, n), (1, 1)).flip(0))


def circulant_operand(n: int, r: int, seed: int, device="cuda", dtype=torch.float64, noise: float = 1e-3):
    """C3: sum_{i<r} diag(d_i) Circ(c_i) + N(0, noise^2), d_i ~ U(0.5, 1.5)."""
    g = _philox([seed, 102, n], device)
    A = noise * torch.randn(n, n, generator=g, device=device, dtype=dtype)
    for _ in range(r):
        d = 0.5 + torch.rand(n, generator=g, device=device, dtype=torch.float64)
        _add_diag_circulant(A, d, smooth_circulant_column(n, g, device))
    return A


def c5_operand(n: int, ncyc: int, r: int, seed: int, operand: int, device="cuda", dtype=torch.float32,
               noise: float = 1e-3):
    """C5: N(0, noise^2) + `ncyc` planted cycles (N(0,1) diagonals) + `r` terms diag(d_i) Circ(c_i).
    n = 32768 fp32 is 4 GiB per operand, so everything is generated in row chunks on the device.
    Returns (A, planted shifts ascending)."""
    g = _philox([seed, 103, n, operand], device)
    A = torch.empty((n, n), device=device, dtype=dtype)
    for s in range(0, n, 2048):
        A[s:s + 2048].normal_(0.0, noise, generator=g)
    J = torch.randperm(n, generator=g, device=device)[:ncyc].tolist()
    i = torch.arange(n, device=device)
    flat = A.view(-1)
    for j in J:
        flat.index_add_(0, i * n + (i - j) % n, torch.randn(n, generator=g, device=device, dtype=dtype))
    for _ in range(r):
        d = 0.5 + torch.rand(n, generator=g, device=device, dtype=torch.float64)
        _add_diag_circulant(A, d, smooth_circulant_column(n, g, device))
    return A, sorted(J)


def c4_operands(n: int, seed: int, device="cuda", k_cyc: int = 64):
    """C4: A = haar-spectrum with sigma_i = (i+1)^-1.5 (fp32), B = N(0, 1e-3^2) + k_cyc N(0,1)
    cycles (fp32), both from one Philox stream keyed by `seed` (the bench / test operands)."""
    g = torch.Generator(device=device).manual_seed(seed)
    sig = (torch.arange(n, device=device, dtype=torch.float64) + 1.0) ** -1.5

    def haar():
        Q, R = torch.linalg.qr(torch.randn(n, n, generator=g, device=device, dtype=torch.float64))
        d = torch.sign(torch.diagonal(R))
        d[d == 0] = 1.0
        return Q * d

    Q1 = haar()
    Q2 = haar()
    A = ((Q1 * sig) @ Q2.T).float().contiguous()
    del Q1, Q2
    B = 1e-3 * torch.randn(n, n, generator=g, device=device, dtype=torch.float32)
    J = torch.randperm(n, generator=g, device=device)[:k_cyc]
    i = torch.arange(n, device=device)
    for j in J.tolist():
        B[i, (i - j) % n] += torch.randn(n, generator=g, device=device, dtype=torch.float32)
    if str(device).startswith("cuda"):
        torch.cuda.synchronize()
    return A, B
