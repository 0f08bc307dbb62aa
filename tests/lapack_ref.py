"""Independent references used to pin the oracle (tests only).

* ``dgbbrd_de``: LAPACK DGBBRD (Givens-based band -> bidiagonal, a different
  algorithm from the paper's Householder bulge chasing) through scipy's
  bundled LAPACK (``scipy.linalg.cython_lapack``), VECT='N', KL=0, KU=b.
* ``gk_right_first``: textbook dense Golub-Kahan Householder bidiagonalisation
  started with a RIGHT reflector on row 0, so that U e1 = V e1 = e1 like the
  bulge-chasing reduction (every right reflector acts on columns >= 1, every
  left one on rows >= 1).  By the Golub-Kahan-Lanczos
  recurrence from v1 = e1, |d| and |e| are then unique.
* ``bidiag_svals``: singular values of upper bidiagonal (d, e) via the
  2n x 2n Golub-Kahan tridiagonal (scipy ``eigvalsh_tridiagonal``).
* ``bidiag_svals_dqds``: the same singular values by LAPACK DLASQ1 (dqds,
  high relative accuracy; seconds at n = 32768 where the GK route takes a
  minute).  Used for the full-size golden comparisons.
"""
from __future__ import annotations

import ctypes

import numpy as np
import scipy.linalg.cython_lapack as _cl
from scipy.linalg import eigvalsh_tridiagonal

_dgbbrd = None


def _get_dgbbrd():
    global _dgbbrd
    if _dgbbrd is None:
        cap = _cl.__pyx_capi__["dgbbrd"]
        ctypes.pythonapi.PyCapsule_GetName.restype = ctypes.c_char_p
        ctypes.pythonapi.PyCapsule_GetName.argtypes = [ctypes.py_object]
        name = ctypes.pythonapi.PyCapsule_GetName(cap)
        ctypes.pythonapi.PyCapsule_GetPointer.restype = ctypes.c_void_p
        ctypes.pythonapi.PyCapsule_GetPointer.argtypes = [ctypes.py_object, ctypes.c_char_p]
        addr = ctypes.pythonapi.PyCapsule_GetPointer(cap, name)
        ip = ctypes.POINTER(ctypes.c_int)
        dp = ctypes.POINTER(ctypes.c_double)
        proto = ctypes.CFUNCTYPE(None, ctypes.c_char_p, ip, ip, ip, ip, ip, dp, ip, dp, dp,
                                 dp, ip, dp, ip, dp, ip, dp, ip)
        _dgbbrd = proto(addr)
    return _dgbbrd


_dlasq1 = None


def _capsule_fn(name, proto):
    cap = _cl.__pyx_capi__[name]
    ctypes.pythonapi.PyCapsule_GetName.restype = ctypes.c_char_p
    ctypes.pythonapi.PyCapsule_GetName.argtypes = [ctypes.py_object]
    nm = ctypes.pythonapi.PyCapsule_GetName(cap)
    ctypes.pythonapi.PyCapsule_GetPointer.restype = ctypes.c_void_p
    ctypes.pythonapi.PyCapsule_GetPointer.argtypes = [ctypes.py_object, ctypes.c_char_p]
    return proto(ctypes.pythonapi.PyCapsule_GetPointer(cap, nm))


def bidiag_svals_dqds(d: np.ndarray, e: np.ndarray) -> np.ndarray:
    """Singular values of the upper bidiagonal (d, e), descending, by LAPACK
    DLASQ1 (dqds).  Signs of d, e do not matter (|d|, |e| are used)."""
    global _dlasq1
    if _dlasq1 is None:
        ip = ctypes.POINTER(ctypes.c_int)
        dp = ctypes.POINTER(ctypes.c_double)
        _dlasq1 = _capsule_fn("dlasq1", ctypes.CFUNCTYPE(None, ip, dp, dp, dp, ip))
    n = len(d)
    if n == 0:
        return np.zeros(0)
    dd = np.abs(np.array(d, dtype=np.float64))
    ee = np.zeros(max(n, 1))
    ee[: n - 1] = np.abs(np.asarray(e, dtype=np.float64)[: n - 1])
    work = np.zeros(4 * n)
    info = ctypes.c_int(0)
    dp = ctypes.POINTER(ctypes.c_double)
    _dlasq1(ctypes.byref(ctypes.c_int(n)), dd.ctypes.data_as(dp), ee.ctypes.data_as(dp),
            work.ctypes.data_as(dp), ctypes.byref(info))
    assert info.value == 0, info.value
    return dd


def dgbbrd_de(band: np.ndarray, b: int):
    """(d, e) from LAPACK DGBBRD on the LAPACK upper band (n, ldband)."""
    f = _get_dgbbrd()
    ab = np.array(band, dtype=np.float64, copy=True, order="C")  # Fortran (ld x n)
    n, ld = ab.shape
    I = ctypes.c_int
    d = np.zeros(n)
    e = np.zeros(max(n - 1, 1))
    dummy = np.zeros(1)
    work = np.zeros(2 * max(n, 1))
    info = I(0)
    dp = ctypes.POINTER(ctypes.c_double)
    f(b"N", ctypes.byref(I(n)), ctypes.byref(I(n)), ctypes.byref(I(0)), ctypes.byref(I(0)),
      ctypes.byref(I(b)), ab.ctypes.data_as(dp), ctypes.byref(I(ld)), d.ctypes.data_as(dp),
      e.ctypes.data_as(dp), dummy.ctypes.data_as(dp), ctypes.byref(I(1)),
      dummy.ctypes.data_as(dp), ctypes.byref(I(1)), dummy.ctypes.data_as(dp),
      ctypes.byref(I(1)), work.ctypes.data_as(dp), ctypes.byref(info))
    assert info.value == 0
    return d, e[: max(n - 1, 0)]


def _house(x):
    alpha = x[0]
    nrm = np.linalg.norm(x)
    v = x.astype(np.float64).copy()
    if nrm == 0.0 or np.all(x[1:] == 0):
        return None, alpha
    beta = -nrm if alpha >= 0 else nrm
    v[0] = alpha - beta
    v /= v[0]
    tau = (beta - alpha) / beta
    return (v, tau), beta


def gk_right_first(A: np.ndarray):
    """Dense Householder bidiagonalisation B = U^T A V, U e1 = V e1 = e1."""
    A = np.array(A, dtype=np.float64, copy=True)
    n = A.shape[0]
    for k in range(n):
        if k > 0:  # left reflector on column k, rows k..n-1
            hv, _ = _house(A[k:, k])
            if hv is not None:
                v, tau = hv
                A[k:, :] -= tau * np.outer(v, v @ A[k:, :])
        if k + 1 < n:  # right reflector on row k, columns k+1..n-1
            hv, _ = _house(A[k, k + 1:])
            if hv is not None:
                v, tau = hv
                A[:, k + 1:] -= tau * np.outer(A[:, k + 1:] @ v, v)
    return np.diag(A).copy(), np.diag(A, 1).copy(), A


def bidiag_svals(d: np.ndarray, e: np.ndarray) -> np.ndarray:
    """Singular values of the upper bidiagonal (d, e), descending."""
    n = len(d)
    if n == 0:
        return np.zeros(0)
    diag = np.zeros(2 * n)
    off = np.zeros(2 * n - 1)
    off[0::2] = d
    if n > 1:
        off[1::2] = e
    w = eigvalsh_tridiagonal(diag, off)
    return np.clip(np.sort(w)[::-1][:n], 0.0, None)
