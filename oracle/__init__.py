"""CPU oracle for Eq. 1 -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import this package.  The
product path (``paper_2101_09808_b200`` and ``libconv.so``) never imports,
links or calls it; the two share no code.  Inputs come from
``paper_2101_09808_b200.inputs`` (seeded generators, no method arithmetic).

Functions and the passage each follows:

* ``conv_eq1``        -- Eq. 1 in Listing 2's loop order
                         (PAPER.md:150-158), double accumulation, plain C
                         (``conv_oracle.c``).  Pinned by tests/test_oracle.py
                         (P1-P9 of SURVEY.md Sec. 8(c)).
* ``conv_eq1_strided`` -- Eq. 1 with stride U (PAPER.md:201 footnote; Table 1,
                         PAPER.md:439, stride-2 layers): In[n,c,U*h+r,U*w+s],
                         explicit input extents, floor output extents; plain C.
                         Pinned by tests/test_oracle.py: U = 1 equals conv_eq1,
                         stride-U output = stride-1 output subsampled (exact),
                         torch conv2d f64 with stride, a hand-worked golden,
                         brute-force points.
* ``conv_eq1_dilated`` -- stride U and dilation D (PAPER.md:201 footnote):
                         In[n,c,U*h+D*r,U*w+D*s]; plain C.  Pinned: D = 1 is
                         conv_eq1_strided; = the strided oracle with a
                         zero-inserted kernel, bit for bit; torch conv2d f64
                         with dilation; brute-force points.
* ``conv_eq1_padded``  -- zero padding (ph, pw) with stride U and dilation D
                         (SURVEY Sec. 8(f) NEXT-2): taps outside the input are
                         skipped; plain C.  Pinned: pad 0 is conv_eq1_dilated;
                         torch conv2d f64 with padding; the interior equals the
                         unpadded output shifted by the pad; all-ones closed
                         form (count of in-range taps); brute-force points.
* ``conv_eq1_point``  -- one output element of Eq. 1 as the correctly rounded
                         sum (``math.fsum``) of its C*R*S exact products; used
                         for sampled parity at full sizes.  Pinned against
                         ``conv_eq1`` and closed forms.
* ``round_bf16_rne``  -- IEEE binary32 -> bfloat16, round-to-nearest-even
                         (bfloat16 = top 16 bits of binary32).
                         reading R5: the BF16 path rounds its inputs this way.
                         Pinned against torch's CPU bf16 cast.
* ``round_tf32_rna``  -- binary32 -> TF32 (10 explicit mantissa bits), round to
                         nearest, ties away from zero.  DESIGN.md reading R5.
                         Pinned by hand-worked tie cases and the half-ulp bound.
"""
from __future__ import annotations

import ctypes
import math
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "conv_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lock = threading.Lock()
_lib = None


def build(force: bool = False) -> str:
    """Compile conv_oracle.c with gcc -O2 -fopenmp (no -ffast-math: the
    double summation must be IEEE round-to-nearest in Listing-2 order)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        cmd = ["gcc", "-O2", "-fPIC", "-shared", "-fopenmp", "-fno-fast-math",
               "-ffp-contract=off", "-o", _LIB, _SRC]
        subprocess.check_call(cmd)
    return _LIB


def _load():
    global _lib
    with _lock:
        if _lib is None:
            build()
            lib = ctypes.CDLL(_LIB)
            lib.oracle_conv_eq1.restype = ctypes.c_int
            lib.oracle_conv_eq1.argtypes = [ctypes.c_int] * 7 + [
                ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int]
            lib.oracle_conv_eq1_strided.restype = ctypes.c_int
            lib.oracle_conv_eq1_strided.argtypes = [ctypes.c_int] * 8 + [
                ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int]
            lib.oracle_conv_eq1_dilated.restype = ctypes.c_int
            lib.oracle_conv_eq1_dilated.argtypes = [ctypes.c_int] * 9 + [
                ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int]
            lib.oracle_conv_eq1_padded.restype = ctypes.c_int
            lib.oracle_conv_eq1_padded.argtypes = [ctypes.c_int] * 11 + [
                ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int]
            lib.oracle_num_threads.restype = ctypes.c_int
            lib.oracle_num_threads.argtypes = [ctypes.c_int]
            _lib = lib
    return _lib


def host_threads() -> int:
    """Threads available to this process (the oracle's default)."""
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:  # pragma: no cover
        return os.cpu_count() or 1


def num_threads(nthreads: int = 0) -> int:
    return _load().oracle_num_threads(nthreads or host_threads())


def conv_eq1(inp: np.ndarray, ker: np.ndarray, nthreads: int = 0) -> np.ndarray:
    """Eq. 1, stride 1, no padding.  ``inp``: fp32 [N,C,H+R-1,W+S-1];
    ``ker``: fp32 [K,C,R,S].  Returns float64 [N,K,H,W]."""
    inp = np.ascontiguousarray(inp, dtype=np.float32)
    ker = np.ascontiguousarray(ker, dtype=np.float32)
    if inp.ndim != 4 or ker.ndim != 4 or inp.shape[1] != ker.shape[1]:
        raise ValueError("expected In [N,C,Hin,Win] and Ker [K,C,R,S] with equal C")
    N, C, Hin, Win = inp.shape
    K, _, R, S = ker.shape
    H, W = Hin - R + 1, Win - S + 1
    if H < 1 or W < 1:
        raise ValueError("input smaller than the kernel")
    out = np.empty((N, K, H, W), dtype=np.float64)
    rc = _load().oracle_conv_eq1(N, K, C, H, W, R, S,
                                 inp.ctypes.data, ker.ctypes.data, out.ctypes.data,
                                 nthreads or host_threads())
    if rc != 0:
        raise ValueError("oracle_conv_eq1 rejected its arguments")
    return out


def conv_eq1_strided(inp: np.ndarray, ker: np.ndarray, stride: int, nthreads: int = 0) -> np.ndarray:
    """Eq. 1 with stride U = ``stride``, no padding.  ``inp``: fp32
    [N,C,Hin,Win]; ``ker``: fp32 [K,C,R,S].  Returns float64 [N,K,H,W] with
    H = (Hin-R)//U + 1, W = (Win-S)//U + 1."""
    inp = np.ascontiguousarray(inp, dtype=np.float32)
    ker = np.ascontiguousarray(ker, dtype=np.float32)
    if inp.ndim != 4 or ker.ndim != 4 or inp.shape[1] != ker.shape[1]:
        raise ValueError("expected In [N,C,Hin,Win] and Ker [K,C,R,S] with equal C")
    N, C, Hin, Win = inp.shape
    K, _, R, S = ker.shape
    if stride < 1 or Hin < R or Win < S:
        raise ValueError("bad stride or input smaller than the kernel")
    H, W = (Hin - R) // stride + 1, (Win - S) // stride + 1
    out = np.empty((N, K, H, W), dtype=np.float64)
    rc = _load().oracle_conv_eq1_strided(N, K, C, Hin, Win, R, S, stride,
                                         inp.ctypes.data, ker.ctypes.data, out.ctypes.data,
                                         nthreads or host_threads())
    if rc != 0:
        raise ValueError("oracle_conv_eq1_strided rejected its arguments")
    return out


def conv_eq1_dilated(inp: np.ndarray, ker: np.ndarray, stride: int, dilation: int, nthreads: int = 0) -> np.ndarray:
    """Eq. 1 with stride U and dilation D, no padding.  ``inp``: fp32
    [N,C,Hin,Win]; ``ker``: fp32 [K,C,R,S].  Returns float64 [N,K,H,W] with
    H = (Hin - D*(R-1) - 1)//U + 1, likewise W."""
    inp = np.ascontiguousarray(inp, dtype=np.float32)
    ker = np.ascontiguousarray(ker, dtype=np.float32)
    if inp.ndim != 4 or ker.ndim != 4 or inp.shape[1] != ker.shape[1]:
        raise ValueError("expected In [N,C,Hin,Win] and Ker [K,C,R,S] with equal C")
    N, C, Hin, Win = inp.shape
    K, _, R, S = ker.shape
    if stride < 1 or dilation < 1 or Hin < dilation * (R - 1) + 1 or Win < dilation * (S - 1) + 1:
        raise ValueError("bad stride/dilation or input smaller than the dilated kernel")
    H = (Hin - dilation * (R - 1) - 1) // stride + 1
    W = (Win - dilation * (S - 1) - 1) // stride + 1
    out = np.empty((N, K, H, W), dtype=np.float64)
    rc = _load().oracle_conv_eq1_dilated(N, K, C, Hin, Win, R, S, stride, dilation,
                                         inp.ctypes.data, ker.ctypes.data, out.ctypes.data,
                                         nthreads or host_threads())
    if rc != 0:
        raise ValueError("oracle_conv_eq1_dilated rejected its arguments")
    return out


def conv_eq1_padded(inp: np.ndarray, ker: np.ndarray, stride: int = 1, dilation: int = 1, padding=0,
                    nthreads: int = 0) -> np.ndarray:
    """Eq. 1 with zero padding ``padding`` (int or (ph, pw)), stride U and
    dilation D.  ``inp``: fp32 [N,C,Hin,Win]; ``ker``: fp32 [K,C,R,S].
    Returns float64 [N,K,H,W], H = (Hin + 2ph - D(R-1) - 1)//U + 1."""
    inp = np.ascontiguousarray(inp, dtype=np.float32)
    ker = np.ascontiguousarray(ker, dtype=np.float32)
    if inp.ndim != 4 or ker.ndim != 4 or inp.shape[1] != ker.shape[1]:
        raise ValueError("expected In [N,C,Hin,Win] and Ker [K,C,R,S] with equal C")
    ph, pw = (padding, padding) if np.isscalar(padding) else padding
    N, C, Hin, Win = inp.shape
    K, _, R, S = ker.shape
    U, D = stride, dilation
    if U < 1 or D < 1 or ph < 0 or pw < 0 or Hin + 2 * ph < D * (R - 1) + 1 or Win + 2 * pw < D * (S - 1) + 1:
        raise ValueError("bad stride/dilation/padding or padded input smaller than the dilated kernel")
    H = (Hin + 2 * ph - D * (R - 1) - 1) // U + 1
    W = (Win + 2 * pw - D * (S - 1) - 1) // U + 1
    out = np.empty((N, K, H, W), dtype=np.float64)
    rc = _load().oracle_conv_eq1_padded(N, K, C, Hin, Win, R, S, U, D, ph, pw,
                                        inp.ctypes.data, ker.ctypes.data, out.ctypes.data, nthreads or host_threads())
    if rc != 0:
        raise ValueError("oracle_conv_eq1_padded rejected its arguments")
    return out


def conv_eq1_point(inp: np.ndarray, ker: np.ndarray, n: int, k: int, h: int, w: int, stride: int = 1,
                   dilation: int = 1, padding=0) -> float:
    """Out[n,k,h,w] of Eq. 1 (stride U, dilation D, zero padding) as the
    correctly rounded sum of its exact products (each fp32*fp32 product is
    exact in float64); taps outside the input contribute nothing."""
    R, S = ker.shape[2], ker.shape[3]
    ph, pw = (padding, padding) if np.isscalar(padding) else padding
    d = dilation
    rows = stride * h + d * np.arange(R) - ph        # input row of tap r
    cols = stride * w + d * np.arange(S) - pw        # input column of tap s
    rk, sk = np.nonzero((rows[:, None] >= 0) & (rows[:, None] < inp.shape[2])
                        & (cols[None, :] >= 0) & (cols[None, :] < inp.shape[3]))
    window = inp[n][:, rows[rk], cols[sk]].astype(np.float64)      # [C, taps in range]
    prods = window * ker[k][:, rk, sk].astype(np.float64)
    return math.fsum(prods.ravel().tolist())


def round_bf16_rne(x: np.ndarray) -> np.ndarray:
    """binary32 -> bfloat16 (round to nearest, ties to even), returned as the
    binary32 value it represents.  bfloat16 keeps the sign, the 8 exponent bits
    and the top 7 mantissa bits of binary32; the discarded low 16 bits are
    rounded: add 0x7FFF plus the lowest kept bit, then truncate.
    NaN handling is out of scope (reading R13)."""
    u = np.ascontiguousarray(x, dtype=np.float32).view(np.uint32).astype(np.uint64)
    lsb = (u >> 16) & 1
    r = ((u + 0x7FFF + lsb) >> 16) << 16
    return (r & 0xFFFFFFFF).astype(np.uint32).view(np.float32)


def round_tf32_rna(x: np.ndarray) -> np.ndarray:
    """binary32 -> TF32 (1 sign, 8 exponent, 10 mantissa bits), round to
    nearest with ties away from zero, returned as binary32.  The discarded low
    13 bits are rounded by adding half of the kept ulp (0x1000) to the
    magnitude and truncating.  NaN handling is out of scope (reading R13)."""
    u = np.ascontiguousarray(x, dtype=np.float32).view(np.uint32).astype(np.uint64)
    r = ((u + 0x1000) >> 13) << 13
    return (r & 0xFFFFFFFF).astype(np.uint32).view(np.float32)
