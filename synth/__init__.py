"""Seeded synthetic input generators shared by the oracle tests, the GPU parity
tests and ``bench.py``.

This module holds NONE of the method's arithmetic (no reflectors, no bulge
chasing): it only draws random banded matrices in the storage layout the
C ABI consumes, and builds the known-spectrum inputs of the paper's accuracy
protocol (PAPER.md §"Numerical Accuracy").  It is imported by both
``oracle``-side tests and product-side code (``bench.py``), and imports
neither of them.

Layout produced everywhere: LAPACK *upper band* storage (``xGBBRD`` with
KL = 0, KU = b; ``xSBTRD`` UPLO='U'), held as a C-contiguous array of shape
``(n, ldband)`` with ``band[j, b + i - j] = A[i, j]`` for
``max(0, j - b) <= i <= j``.  Column ``j`` of the Fortran band is row ``j`` of
the numpy array, so ``band.ravel()`` is exactly the Fortran column-major
buffer with leading dimension ``ldband``.  Unused corner slots are 0.

Input recipe: i.i.d. N(0, 1) entries on
the band (0 <= j - i <= b), zero elsewhere, drawn from numpy's counter-based
Philox generator keyed by (seed, matrix_id), in fp64, then rounded to the
requested dtype with round-to-nearest-even.
"""
from __future__ import annotations

import numpy as np

DTYPES = {"f16": np.float16, "f32": np.float32, "f64": np.float64}


def _rng(seed: int, matrix_id: int) -> np.random.Generator:
    return np.random.Generator(np.random.Philox(key=[int(seed) & (2**64 - 1), int(matrix_id) & (2**64 - 1)]))


def random_band(n: int, b: int, dtype: str = "f64", seed: int = 0, matrix_id: int = 0,
                ldband: int | None = None) -> np.ndarray:
    """One n x n upper-banded matrix with i.i.d. N(0,1) band entries.

    Returns the LAPACK upper-band array of shape (n, ldband) in ``dtype``.
    ``b`` is clamped to n - 1 for the draw (entries beyond the matrix do not
    exist); the array still has ``ldband >= b + 1`` slots per column.
    """
    if ldband is None:
        ldband = b + 1
    if ldband < b + 1:
        raise ValueError("ldband < b + 1")
    npdt = DTYPES[dtype]
    out = np.zeros((n, ldband), dtype=np.float64)
    if n == 0:
        return out.astype(npdt)
    bb = min(b, n - 1)
    g = _rng(seed, matrix_id)
    # draw column by column in a fixed order: offsets 0..bb (k = j - i)
    vals = g.standard_normal((n, bb + 1))  # vals[j, k] = A[j - k, j]
    for k in range(bb + 1):
        # slot b + i - j = b - k ; valid for j >= k
        out[k:, b - k] = vals[k:, k]
    return out.astype(npdt)


def random_band_batch(batch: int, n: int, b: int, dtype: str = "f64", seed: int = 0,
                      first_id: int = 0, ldband: int | None = None) -> np.ndarray:
    """``batch`` independent matrices, matrix ids first_id .. first_id+batch-1.

    Shape (batch, n, ldband); matrix k equals ``random_band(..., matrix_id=first_id+k)``.
    """
    if ldband is None:
        ldband = b + 1
    out = np.empty((batch, n, ldband), dtype=DTYPES[dtype])
    for k in range(batch):
        out[k] = random_band(n, b, dtype, seed, first_id + k, ldband)
    return out


def band_to_dense(band: np.ndarray, b: int) -> np.ndarray:
    """Expand LAPACK upper-band storage (n, ldband) into a dense fp64 n x n matrix."""
    n = band.shape[0]
    A = np.zeros((n, n), dtype=np.float64)
    for j in range(n):
        for i in range(max(0, j - b), j + 1):
            A[i, j] = float(band[j, b + i - j])
    return A


def dense_to_band(A: np.ndarray, b: int, dtype: str = "f64", ldband: int | None = None) -> np.ndarray:
    """Pack the upper band (0 <= j - i <= b) of a dense matrix; raises if A is not banded."""
    n = A.shape[0]
    if A.shape != (n, n):
        raise ValueError("not square")
    if ldband is None:
        ldband = b + 1
    iu = np.triu_indices(n, b + 1)
    il = np.tril_indices(n, -1)
    if np.any(A[iu] != 0) or np.any(A[il] != 0):
        raise ValueError("matrix is not upper-banded with bandwidth b")
    out = np.zeros((n, ldband), dtype=np.float64)
    for j in range(n):
        for i in range(max(0, j - b), j + 1):
            out[j, b + i - j] = A[i, j]
    return out.astype(DTYPES[dtype])


# ---------------------------------------------------------------------------
# Known-spectrum inputs (paper accuracy protocol)
# ---------------------------------------------------------------------------

def spectrum(kind: str, n: int, seed: int = 0) -> np.ndarray:
    """Prescribed singular values in [0, 1]: 'arith' (uniform spacing),
    'log' (logarithmic decay) or 'qcirc' (quarter-circle distribution)."""
    if kind == "arith":
        s = np.linspace(1.0, 1.0 / n, n)
    elif kind == "log":
        s = np.logspace(0.0, -6.0, n)
    elif kind == "qcirc":
        # quantiles of the quarter-circle law on [0, 1]: density (4/pi) sqrt(1-x^2)
        # CDF F(x) = (2/pi)(x sqrt(1-x^2) + asin x); invert by bisection
        u = (np.arange(n) + 0.5) / n
        lo, hi = np.zeros(n), np.ones(n)
        for _ in range(60):
            mid = 0.5 * (lo + hi)
            F = (2.0 / np.pi) * (mid * np.sqrt(1.0 - mid * mid) + np.arcsin(mid))
            lo = np.where(F < u, mid, lo)
            hi = np.where(F < u, hi, mid)
        s = np.sort(0.5 * (lo + hi))[::-1].copy()
    else:
        raise ValueError(kind)
    return s


def known_spectrum_dense(n: int, sigma: np.ndarray, seed: int = 0) -> np.ndarray:
    """A = U diag(sigma) V^T with Haar-like U, V from QR of Gaussian matrices."""
    g = _rng(seed, 10_000_019)
    U, R = np.linalg.qr(g.standard_normal((n, n)))
    U = U * np.sign(np.diag(R))
    V, R = np.linalg.qr(g.standard_normal((n, n)))
    V = V * np.sign(np.diag(R))
    return (U * sigma) @ V.T


def dense_to_upper_band(A: np.ndarray, b: int) -> np.ndarray:
    """Stage 1 (test-side only): classical block Householder reduction of a
    dense matrix to upper-banded form with b superdiagonals ("first
    reduced to banded form using the classical block Householder reduction").

    For k = 0, b, 2b, ...: QR of the column panel A[k:, k:k+b] (left
    orthogonal transform) then LQ of the row panel A[k:k+b, k+b:] (right
    orthogonal transform).  Eliminated entries are set to exact 0.
    Returns a dense fp64 matrix with the same singular values as A.
    """
    A = np.array(A, dtype=np.float64, copy=True)
    n = A.shape[0]
    for k in range(0, n, b):
        kb = min(k + b, n)
        Q, _ = np.linalg.qr(A[k:, k:kb], mode="complete")
        A[k:, k:] = Q.T @ A[k:, k:]
        for jj in range(k, kb):
            A[jj + 1:, jj] = 0.0
        if kb < n:
            Q2, _ = np.linalg.qr(A[k:kb, kb:].T, mode="complete")
            A[:, kb:] = A[:, kb:] @ Q2
            for ii in range(k, kb):
                A[ii, kb + (ii - k) + 1:] = 0.0
    return A
