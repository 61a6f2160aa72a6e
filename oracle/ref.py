"""ORACLE — TEST INFRASTRUCTURE ONLY. ctypes binding of oracle/ffs_ref.c (libffs_ref.so).

Functions mirror the C-ABI semantics of the CUDA library on HOST numpy arrays
(SURVEY.md §8b "Oracle mirror"): positions are 0-based, in sampling order.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "libffs_ref.so")
_SRC = [os.path.join(_HERE, "ffs_ref.c"), os.path.join(_HERE, "ffs_ref_core.h")]
_lib = None

F64, C128 = 0, 1


def build(force: bool = False) -> str:
    """Compile libffs_ref.so with gcc (-O2, IEEE semantics, OpenMP across samples)."""
    stale = (not os.path.exists(_SO)) or any(os.path.getmtime(s) > os.path.getmtime(_SO) for s in _SRC)
    if force or stale:
        tmp = _SO + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-fopenmp", "-shared", "-fPIC", "-o", tmp,
                               _SRC[0], "-lm"], cwd=_HERE)
        os.replace(tmp, _SO)
    return _SO


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_SO)
        i64, i32p, f64p, vp = ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p
        L.ffs_ref_sample_marginal.argtypes = [vp, i64, i64, ctypes.c_int, i64, i64, vp, vp, vp, ctypes.c_int]
        L.ffs_ref_sample.argtypes = [vp, i64, i64, ctypes.c_int, i64, vp, vp, vp, ctypes.c_int]
        L.ffs_ref_weights.argtypes = [vp, i64, i64, ctypes.c_int, i64, i64, vp, vp, vp]
        L.ffs_ref_chain.argtypes = [vp, i64, i64, ctypes.c_int, i64, vp, vp, vp, vp, vp]
        L.ffs_ref_permutation.argtypes = [vp, i64, i64, vp]
        L.ffs_ref_permutation.restype = None
        L.ffs_ref_occupation.argtypes = [vp, i64, i64, i64, vp]
        L.ffs_ref_pair_occupation.argtypes = [vp, i64, i64, i64, vp]
        L.ffs_ref_gutzwiller.argtypes = [vp, i64, i64, i64, ctypes.c_double, vp]
        L.ffs_ref_sample_metropolis.argtypes = [vp, i64, i64, ctypes.c_int, i64, i64, i64, vp, vp, vp, vp,
                                                ctypes.c_int]
        L.ffs_ref_sample_hkpv.argtypes = [vp, i64, i64, ctypes.c_int, i64, i64, vp, vp, vp, i64, vp, vp,
                                          ctypes.c_int]
        L.ffs_ref_sample_lensemble.argtypes = [vp, vp, i64, i64, ctypes.c_int, i64, vp, vp, vp, vp, ctypes.c_int]
        L.ffs_ref_num_threads.restype = ctypes.c_int
        _lib = L
    return _lib


def _ptr(a):
    return None if a is None else a.ctypes.data


def _u_bytes(U):
    U = np.ascontiguousarray(U)
    if np.iscomplexobj(U):
        return np.ascontiguousarray(U.astype(np.complex128)), C128
    return np.ascontiguousarray(U.astype(np.float64)), F64


def permutation(u, N, Np=None):
    u = np.ascontiguousarray(u, dtype=np.float64)
    Np = N if Np is None else Np
    m = np.empty(N, dtype=np.int32)
    lib().ffs_ref_permutation(_ptr(u), N, Np, _ptr(m))
    return m


def sample(U, uniforms, Np=None, nthreads=0, return_flags=False):
    """M samples from uniforms [M][2Np]; returns positions [M][Np] int32 (and flags)."""
    Ub, dt = _u_bytes(U)
    L, N = Ub.shape
    Np = N if Np is None else Np
    uni = np.ascontiguousarray(uniforms, dtype=np.float64)
    M = uni.shape[0]
    assert uni.shape == (M, 2 * Np), (uni.shape, Np)
    pos = np.empty((M, Np), dtype=np.int32)
    flags = np.empty(M, dtype=np.int32)
    rc = lib().ffs_ref_sample_marginal(_ptr(Ub), L, N, dt, M, Np, _ptr(uni), _ptr(pos), _ptr(flags), nthreads)
    if rc != 0:
        raise ValueError(f"ffs_ref_sample_marginal rc={rc}")
    return (pos, flags) if return_flags else pos


def weights(U, uniforms, Np=None):
    """Positions [S][Np] and normalised conditional weights [S][Np][L] for the rows of uniforms."""
    Ub, dt = _u_bytes(U)
    L, N = Ub.shape
    Np = N if Np is None else Np
    uni = np.ascontiguousarray(uniforms, dtype=np.float64)
    S = uni.shape[0]
    pos = np.empty((S, Np), dtype=np.int32)
    w = np.empty((S, Np, L), dtype=np.float64)
    rc = lib().ffs_ref_weights(_ptr(Ub), L, N, dt, S, Np, _ptr(uni), _ptr(pos), _ptr(w))
    if rc != 0:
        raise ValueError(f"ffs_ref_weights rc={rc}")
    return pos, w


def chain(U, m, x):
    """Teacher-forced chain: (weights [Np][L], hnorm2 [Np], totals [Np]) for permutation m, positions x."""
    Ub, dt = _u_bytes(U)
    L, N = Ub.shape
    m = np.ascontiguousarray(m, dtype=np.int32)
    x = np.ascontiguousarray(x, dtype=np.int32)
    Np = x.shape[0]
    w = np.empty((Np, L), dtype=np.float64)
    hn2 = np.empty(Np, dtype=np.float64)
    tot = np.empty(Np, dtype=np.float64)
    rc = lib().ffs_ref_chain(_ptr(Ub), L, N, dt, Np, _ptr(m), _ptr(x), _ptr(w), _ptr(hn2), _ptr(tot))
    if rc != 0:
        raise ValueError(f"ffs_ref_chain rc={rc}")
    return w, hn2, tot


def sample_lensemble(V, lam, uniforms, nthreads=0):
    """L-ensemble DPP: eigenvector j kept iff u_j < lambda_j/(lambda_j+1), then FFS
    on the kept columns. uniforms [M][3K]; returns positions [M][K] (-1 padded), counts [M], flags [M]."""
    Vb, dt = _u_bytes(V)
    L, K = Vb.shape
    lam = np.ascontiguousarray(lam, dtype=np.float64)
    uni = np.ascontiguousarray(uniforms, dtype=np.float64)
    M = uni.shape[0]
    assert lam.shape == (K,) and uni.shape == (M, 3 * K), (lam.shape, uni.shape)
    pos = np.empty((M, K), dtype=np.int32)
    cnt = np.empty(M, dtype=np.int32)
    flags = np.empty(M, dtype=np.int32)
    rc = lib().ffs_ref_sample_lensemble(_ptr(Vb), _ptr(lam), L, K, dt, M, _ptr(uni), _ptr(pos), _ptr(cnt),
                                        _ptr(flags), nthreads)
    if rc != 0:
        raise ValueError(f"ffs_ref_sample_lensemble rc={rc}")
    return pos, cnt, flags


def occupation(positions, L):
    """occ[x] = number of samples with site x occupied (entries < 0 skipped)."""
    pos = np.ascontiguousarray(positions, dtype=np.int32)
    occ = np.empty(L, dtype=np.uint64)
    assert lib().ffs_ref_occupation(_ptr(pos), pos.shape[0], pos.shape[1], L, _ptr(occ)) == 0
    return occ


def pair_occupation(positions, W):
    """pair[x][y] = number of samples with x and y occupied (x, y < W)."""
    pos = np.ascontiguousarray(positions, dtype=np.int32)
    pair = np.empty((W, W), dtype=np.uint64)
    assert lib().ffs_ref_pair_occupation(_ptr(pos), pos.shape[0], pos.shape[1], W, _ptr(pair)) == 0
    return pair


def gutzwiller(positions, L, V):
    """Gutzwiller reweighting (Supp S5) of spinful samples (rows 2s up, 2s+1 down):
    [<J^2>_0, <D>_J, <n_0>_J .. <n_{L-1}>_J] with J^2 = exp(-V D)."""
    pos = np.ascontiguousarray(positions, dtype=np.int32)
    assert pos.shape[0] % 2 == 0
    res = np.empty(2 + L, dtype=np.float64)
    assert lib().ffs_ref_gutzwiller(_ptr(pos), pos.shape[0] // 2, pos.shape[1], L, float(V), _ptr(res)) == 0
    return res


def sample_metropolis(U, uniforms, Np, Mc, nthreads=0, return_margins=False):
    """Supp S7 variant: Mc Metropolis updates per step with uniform discrete
    proposals. uniforms [M][Np + Np (1 + 2 Mc)]; returns positions [M][Np], flags [M] (and the
    per-step decision margins [M][Np])."""
    Ub, dt = _u_bytes(U)
    L, N = Ub.shape
    uni = np.ascontiguousarray(uniforms, dtype=np.float64)
    M = uni.shape[0]
    assert uni.shape == (M, Np + Np * (1 + 2 * Mc)), (uni.shape, Np, Mc)
    pos = np.empty((M, Np), dtype=np.int32)
    flags = np.empty(M, dtype=np.int32)
    mg = np.empty((M, Np), dtype=np.float64) if return_margins else None
    rc = lib().ffs_ref_sample_metropolis(_ptr(Ub), L, N, dt, M, Np, Mc, _ptr(uni), _ptr(pos), _ptr(flags), _ptr(mg),
                                         nthreads)
    if rc != 0:
        raise ValueError(f"ffs_ref_sample_metropolis rc={rc}")
    return (pos, flags, mg) if return_margins else (pos, flags)


def sample_hkpv(U, uniforms, Np=None, S=0, nthreads=0):
    """Modified HKPV sampler (the paper's comparator).
    uniforms [M][Np] selection draws. Returns positions [M][Np], flags [M], and for S > 0 the
    normalised weights [S][Np][L] and totals [S][Np] of the first S samples."""
    Ub, dt = _u_bytes(U)
    L, N = Ub.shape
    uni = np.ascontiguousarray(uniforms, dtype=np.float64)
    M = uni.shape[0]
    Np = uni.shape[1] if Np is None else Np
    assert uni.shape == (M, Np), (uni.shape, Np)
    pos = np.empty((M, Np), dtype=np.int32)
    flags = np.empty(M, dtype=np.int32)
    w = np.empty((S, Np, L), dtype=np.float64) if S else None
    tot = np.empty((S, Np), dtype=np.float64) if S else None
    rc = lib().ffs_ref_sample_hkpv(_ptr(Ub), L, N, dt, M, Np, _ptr(uni), _ptr(pos), _ptr(flags), S, _ptr(w),
                                   _ptr(tot), nthreads)
    if rc != 0:
        raise ValueError(f"ffs_ref_sample_hkpv rc={rc}")
    return (pos, flags, w, tot) if S else (pos, flags)


def num_threads() -> int:
    return int(lib().ffs_ref_num_threads())
