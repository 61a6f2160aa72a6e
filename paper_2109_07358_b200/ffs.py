"""Thin Python binding of libffs.so (include/ffs.h): argument marshalling only.

Every step of the sampling path runs in the CUDA kernels of the library; PyTorch provides
device memory and streams. If the library is missing this module raises — there is no CPU
fallback.
"""
from __future__ import annotations

import ctypes
import os
from typing import Optional, Tuple

import torch

from . import build as _build

FFS_F64, FFS_C128 = 0, 1
FFS_OK, FFS_EINVAL, FFS_ECUDA, FFS_ENOWS = 0, -1, -2, -3

# include/ffs.h ffs_option
OPTIONS = {
    "dense_gemm": 1,        # 8 = Ozaki int8 x 8 slices (default), 7 = 7 slices, 0 = DMMA
    "dense_theta": 2,       # gathered/GEMM crossover fraction (< 0: default)
    "dense_batch": 3,       # samples per lockstep batch (0: default)
    "block_step": 4,        # 1: large-L block-step paths (default); 0: per-sample cluster kernel
    "large_l_marginal": 5,  # 1: large-L marginals on the block-step kernels (default)
    "cluster": 6,           # 1: L >= 2048 on cluster kernels (default); 0: one CTA per sample
    "graph": 7,             # 1: block-step launches replayed as a CUDA graph (default)
    "force_generic": 8,     # 1: every shape on the per-sample warp/CTA-owner kernel
    "gemm_2sm": 9,          # 1: the 8-slice Ozaki GEMM as tcgen05 CTA pairs, 256x128 two-pass tiles (default); 3: 256x64
    "gram_draw": 10,        # 1: GEMM block steps draw on the tile Gram matrices (default)
    "gram_kappa": 11,       # cancellation guard of the Gram draws (default 1e4)
    "dense_min_l": 12,      # smallest L on the block-step paths (default 2048)
    "dense_min_n": 13,      # smallest N on the block-step paths (default 256)
    "tile_gram": 14,        # 1: small-N' real shapes on the tile-Gram path (default)
    "gj_pair": 15,          # 1: two blocks' trailing Gauss-Jordan updates in one pass (default)
}

EXPORTED = (
    "ffs_workspace_bytes",
    "ffs_sample",
    "ffs_sample_marginal",
    "ffs_debug_trace",
    "ffs_host_workspace_bytes",
    "ffs_sample_host",
    "ffs_last_launch_count",
    "ffs_profile_enable",
    "ffs_last_kernel_ms",
    "ffs_lensemble_workspace_bytes",
    "ffs_sample_lensemble",
    "ffs_metropolis_workspace_bytes",
    "ffs_sample_metropolis",
    "ffs_hkpv_workspace_bytes",
    "ffs_sample_hkpv",
    "ffs_occupation",
    "ffs_pair_occupation",
    "ffs_gutzwiller_workspace_bytes",
    "ffs_gutzwiller_reweight",
    "ffs_set_option",
    "ffs_get_option",
    "ffs_gram_counters",
    "ffs_last_error",
)

_lib = None


class FFSError(RuntimeError):
    pass


def lib_path() -> str:
    """libffs.so in the package directory; FFS_LIBRARY=checked selects the bounds-checked build
    (libffs_checked.so, -DFFS_CHECKED) for the checked test runs."""
    return _build.SO_CHECKED if os.environ.get("FFS_LIBRARY") == "checked" else _build.SO


def load(build_if_missing: bool = True):
    """Load libffs.so (building it in-tree with nvcc if it is missing and nvcc exists)."""
    global _lib
    if _lib is not None:
        return _lib
    so = lib_path()
    if not os.path.exists(so):
        if not build_if_missing:
            raise FFSError(f"{so} missing: run python -m paper_2109_07358_b200.build")
        _build.build(checked=so == _build.SO_CHECKED)
    L = ctypes.CDLL(so)
    i64, vp, sz = ctypes.c_int64, ctypes.c_void_p, ctypes.c_size_t
    ci = ctypes.c_int
    L.ffs_workspace_bytes.argtypes = [i64, i64, i64, ci, i64]
    L.ffs_workspace_bytes.restype = sz
    L.ffs_sample.argtypes = [vp, i64, i64, ci, i64, vp, vp, vp, vp, sz, vp]
    L.ffs_sample_marginal.argtypes = [vp, i64, i64, ci, i64, i64, vp, vp, vp, vp, sz, vp]
    L.ffs_debug_trace.argtypes = [vp, i64, i64, ci, i64, i64, vp, vp, vp, vp, sz, vp, i64, i64, vp]
    L.ffs_host_workspace_bytes.argtypes = [i64, i64, i64, ci, i64]
    L.ffs_host_workspace_bytes.restype = sz
    L.ffs_sample_host.argtypes = [vp, i64, i64, ci, i64, i64, vp, vp, vp, vp, sz, vp]
    L.ffs_last_launch_count.restype = ci
    L.ffs_profile_enable.argtypes = [ci]
    L.ffs_last_kernel_ms.restype = ctypes.c_float
    L.ffs_lensemble_workspace_bytes.argtypes = [i64, i64, ci, i64]
    L.ffs_lensemble_workspace_bytes.restype = sz
    L.ffs_sample_lensemble.argtypes = [vp, vp, i64, i64, ci, i64, vp, vp, vp, vp, vp, sz, vp]
    L.ffs_metropolis_workspace_bytes.argtypes = [i64, i64, i64, i64, ci, i64]
    L.ffs_metropolis_workspace_bytes.restype = sz
    L.ffs_sample_metropolis.argtypes = [vp, i64, i64, ci, i64, i64, i64, vp, vp, vp, vp, sz, vp]
    L.ffs_hkpv_workspace_bytes.argtypes = [i64, i64, i64, ci, i64]
    L.ffs_hkpv_workspace_bytes.restype = sz
    L.ffs_sample_hkpv.argtypes = [vp, i64, i64, ci, i64, i64, vp, vp, vp, vp, sz, vp]
    L.ffs_occupation.argtypes = [vp, i64, i64, i64, vp, vp]
    L.ffs_pair_occupation.argtypes = [vp, i64, i64, i64, vp, vp]
    L.ffs_gutzwiller_workspace_bytes.argtypes = [i64, i64]
    L.ffs_gutzwiller_workspace_bytes.restype = sz
    L.ffs_gutzwiller_reweight.argtypes = [vp, i64, i64, i64, ctypes.c_double, vp, vp, vp, sz, vp]
    L.ffs_set_option.argtypes = [ci, ctypes.c_double]
    L.ffs_get_option.argtypes = [ci]
    L.ffs_get_option.restype = ctypes.c_double
    L.ffs_gram_counters.argtypes = [vp, ci]
    L.ffs_last_error.restype = ctypes.c_char_p
    _lib = L
    return L


def _check(rc: int):
    if rc != FFS_OK:
        msg = load().ffs_last_error().decode()
        raise FFSError(f"libffs rc={rc}: {msg}")


def _dtype_code(U: torch.Tensor) -> int:
    if U.dtype == torch.float64:
        return FFS_F64
    if U.dtype == torch.complex128:
        return FFS_C128
    raise FFSError(f"U must be float64 or complex128, got {U.dtype}")


def _stream_handle(stream: Optional[torch.cuda.Stream], device) -> int:
    s = stream if stream is not None else torch.cuda.current_stream(device)
    return s.cuda_stream


def ffs_workspace_bytes(L: int, N: int, Nprime: int, dtype: int, M: int) -> int:
    return int(load().ffs_workspace_bytes(L, N, Nprime, dtype, M))


def ffs_host_workspace_bytes(L: int, N: int, Nprime: int, dtype: int, M: int) -> int:
    return int(load().ffs_host_workspace_bytes(L, N, Nprime, dtype, M))


def ffs_last_launch_count() -> int:
    return int(load().ffs_last_launch_count())


def ffs_profile_enable(on: bool = True) -> None:
    load().ffs_profile_enable(1 if on else 0)


def ffs_last_kernel_ms() -> float:
    return float(load().ffs_last_kernel_ms())


def ffs_gram_counters(reset: bool = False):
    """ffs_gram_counters (include/ffs.h): (draws, direct recomputations) of the Gram draw kernel."""
    out = (ctypes.c_ulonglong * 2)()
    _check(load().ffs_gram_counters(ctypes.cast(out, ctypes.c_void_p), 1 if reset else 0))
    return int(out[0]), int(out[1])


def set_option(name: str, value: float) -> None:
    """ffs_set_option (include/ffs.h): a NaN value restores the default."""
    _check(load().ffs_set_option(OPTIONS[name], float(value)))


def get_option(name: str) -> float:
    return float(load().ffs_get_option(OPTIONS[name]))


def reset_options() -> None:
    for name in OPTIONS:
        set_option(name, float("nan"))


class Workspace:
    """Caller-owned device workspace (torch allocation), grown on demand."""

    def __init__(self, device="cuda"):
        self.device = torch.device(device)
        self.buf = None

    def get(self, nbytes: int) -> Tuple[int, int]:
        if nbytes == 0:
            return 0, 0
        if self.buf is None or self.buf.numel() < nbytes:
            self.buf = torch.empty(nbytes, dtype=torch.uint8, device=self.device)
        return self.buf.data_ptr(), self.buf.numel()


def _check_out(t: Optional[torch.Tensor], shape, name: str, cuda: bool):
    """Caller-supplied outputs: int32, contiguous, the exact shape, on the right side."""
    if t is None:
        return
    if t.dtype != torch.int32 or tuple(t.shape) != tuple(shape) or not t.is_contiguous() or t.is_cuda != cuda:
        where = "CUDA" if cuda else "host"
        raise FFSError(f"{name} must be a contiguous int32 {where} tensor of shape {tuple(shape)}, "
                       f"got {t.dtype} {tuple(t.shape)} on {t.device}")


def _keep_alive(stream, *tensors):
    """The library works asynchronously on `stream`: tell the caching allocator that these
    tensors (temporaries included) are in use there, so their memory is not handed to other work
    on torch's current stream before the kernels finish."""
    if stream is None:
        return
    for t in tensors:
        if t is not None and t.is_cuda:
            t.record_stream(stream)


def _prep(U: torch.Tensor, uniforms: torch.Tensor, Nprime: int):
    if not (U.is_cuda and uniforms.is_cuda):
        raise FFSError("U and uniforms must be CUDA tensors (use ffs_sample_host for host buffers)")
    if U.dim() != 2:
        raise FFSError("U must be 2-D [L][N]")
    U = U.contiguous()
    uniforms = uniforms.contiguous()
    if uniforms.dtype != torch.float64 or uniforms.dim() != 2 or uniforms.shape[1] != 2 * Nprime:
        raise FFSError(f"uniforms must be float64 [M][2N'] with N'={Nprime}, got {tuple(uniforms.shape)}")
    return U, uniforms


def ffs_sample_marginal(U: torch.Tensor, uniforms: torch.Tensor, Nprime: int,
                        positions: Optional[torch.Tensor] = None, flags: Optional[torch.Tensor] = None,
                        workspace: Optional[Workspace] = None, stream=None, with_flags: bool = False):
    """Device path: positions int32 [M][N'] (and flags int32 [M] if with_flags)."""
    U, uniforms = _prep(U, uniforms, Nprime)
    L, N = U.shape
    M = uniforms.shape[0]
    dt = _dtype_code(U)
    _check_out(positions, (M, Nprime), "positions", True)
    _check_out(flags, (M,), "flags", True)
    if positions is None:
        positions = torch.empty((M, Nprime), dtype=torch.int32, device=U.device)
    if flags is None and with_flags:
        flags = torch.empty(M, dtype=torch.int32, device=U.device)
    ws = workspace if workspace is not None else Workspace(U.device)
    need = ffs_workspace_bytes(L, N, Nprime, dt, M)
    if need == 0 and M > 0:
        _check(load().ffs_sample_marginal(U.data_ptr(), L, N, dt, M, Nprime, None, None, None, None, 0, None))
    wp, wn = ws.get(need)
    rc = load().ffs_sample_marginal(U.data_ptr(), L, N, dt, M, Nprime, uniforms.data_ptr(), positions.data_ptr(),
                                    flags.data_ptr() if flags is not None else None, wp, wn,
                                    _stream_handle(stream, U.device))
    _check(rc)
    _keep_alive(stream, U, uniforms, positions, flags, ws.buf)
    return (positions, flags) if with_flags else positions


def ffs_sample(U: torch.Tensor, uniforms: torch.Tensor, positions: Optional[torch.Tensor] = None,
               flags: Optional[torch.Tensor] = None, workspace: Optional[Workspace] = None, stream=None,
               with_flags: bool = False):
    """Device path, full sampling (N' = N): positions int32 [M][N]."""
    N = U.shape[1]
    U, uniforms = _prep(U, uniforms, N)
    L = U.shape[0]
    M = uniforms.shape[0]
    dt = _dtype_code(U)
    _check_out(positions, (M, N), "positions", True)
    _check_out(flags, (M,), "flags", True)
    if positions is None:
        positions = torch.empty((M, N), dtype=torch.int32, device=U.device)
    if flags is None and with_flags:
        flags = torch.empty(M, dtype=torch.int32, device=U.device)
    ws = workspace if workspace is not None else Workspace(U.device)
    wp, wn = ws.get(ffs_workspace_bytes(L, N, N, dt, M))
    rc = load().ffs_sample(U.data_ptr(), L, N, dt, M, uniforms.data_ptr(), positions.data_ptr(),
                           flags.data_ptr() if flags is not None else None, wp, wn,
                           _stream_handle(stream, U.device))
    _check(rc)
    _keep_alive(stream, U, uniforms, positions, flags, ws.buf)
    return (positions, flags) if with_flags else positions


def ffs_debug_trace(U: torch.Tensor, uniforms: torch.Tensor, Nprime: int, S: int, S0: int = 0,
                    workspace: Optional[Workspace] = None, stream=None):
    """Positions [M][N'], flags [M] and normalised weights [S][N'][L] of samples S0 .. S0+S-1."""
    U, uniforms = _prep(U, uniforms, Nprime)
    L, N = U.shape
    M = uniforms.shape[0]
    dt = _dtype_code(U)
    S = max(0, min(S, M - S0))
    positions = torch.empty((M, Nprime), dtype=torch.int32, device=U.device)
    flags = torch.empty(M, dtype=torch.int32, device=U.device)
    weights = torch.zeros((S, Nprime, L), dtype=torch.float64, device=U.device)
    ws = workspace if workspace is not None else Workspace(U.device)
    wp, wn = ws.get(ffs_workspace_bytes(L, N, Nprime, dt, M))
    rc = load().ffs_debug_trace(U.data_ptr(), L, N, dt, M, Nprime, uniforms.data_ptr(), positions.data_ptr(),
                                flags.data_ptr(), wp, wn, _stream_handle(stream, U.device), S0, S,
                                weights.data_ptr())
    _check(rc)
    _keep_alive(stream, U, uniforms, positions, flags, weights, ws.buf)
    return positions, flags, weights


def ffs_sample_host(U: torch.Tensor, uniforms: torch.Tensor, Nprime: int,
                    positions: Optional[torch.Tensor] = None, flags: Optional[torch.Tensor] = None,
                    workspace: Optional[Workspace] = None, stream=None, device="cuda"):
    """End-to-end path on HOST tensors (pinned recommended): H2D, sampling, D2H inside the call."""
    if U.is_cuda or uniforms.is_cuda:
        raise FFSError("ffs_sample_host takes host tensors")
    U = U.contiguous()
    uniforms = uniforms.contiguous()
    L, N = U.shape
    M = uniforms.shape[0]
    dt = _dtype_code(U)
    if uniforms.dtype != torch.float64 or uniforms.dim() != 2 or uniforms.shape[1] != 2 * Nprime:
        raise FFSError(f"uniforms must be float64 [M][2N'] with N'={Nprime}, got {tuple(uniforms.shape)}")
    _check_out(positions, (M, Nprime), "positions", False)
    _check_out(flags, (M,), "flags", False)
    if positions is None:
        positions = torch.empty((M, Nprime), dtype=torch.int32, pin_memory=True)
    ws = workspace if workspace is not None else Workspace(device)
    wp, wn = ws.get(ffs_host_workspace_bytes(L, N, Nprime, dt, M))
    rc = load().ffs_sample_host(U.data_ptr(), L, N, dt, M, Nprime, uniforms.data_ptr(), positions.data_ptr(),
                                flags.data_ptr() if flags is not None else None, wp, wn,
                                _stream_handle(stream, ws.device))
    _check(rc)
    return positions


def ffs_sample_lensemble(V: torch.Tensor, lam: torch.Tensor, uniforms: torch.Tensor,
                         workspace: Optional[Workspace] = None, stream=None):
    """L-ensemble DPP: eigenvector j of C kept iff u_j < lam_j/(lam_j+1), then
    FFS on the kept columns. V [L][K] (float64/complex128), lam [K] float64, uniforms [M][3K].
    Returns positions int32 [M][K] (-1 past N_i), counts int32 [M], flags int32 [M]."""
    if not (V.is_cuda and lam.is_cuda and uniforms.is_cuda):
        raise FFSError("V, lam and uniforms must be CUDA tensors")
    if V.dim() != 2:
        raise FFSError("V must be 2-D [L][K]")
    V = V.contiguous()
    L, K = V.shape
    lam = lam.contiguous()
    uniforms = uniforms.contiguous()
    if lam.dtype != torch.float64 or tuple(lam.shape) != (K,):
        raise FFSError(f"lam must be float64 [K={K}]")
    if uniforms.dtype != torch.float64 or uniforms.dim() != 2 or uniforms.shape[1] != 3 * K:
        raise FFSError(f"uniforms must be float64 [M][3K] with K={K}, got {tuple(uniforms.shape)}")
    M = uniforms.shape[0]
    dt = _dtype_code(V)
    positions = torch.empty((M, K), dtype=torch.int32, device=V.device)
    counts = torch.empty(M, dtype=torch.int32, device=V.device)
    flags = torch.empty(M, dtype=torch.int32, device=V.device)
    ws = workspace if workspace is not None else Workspace(V.device)
    need = int(load().ffs_lensemble_workspace_bytes(L, K, dt, M))
    if need == 0 and M > 0:
        _check(load().ffs_sample_lensemble(V.data_ptr(), lam.data_ptr(), L, K, dt, M, None, None, None, None,
                                           None, 0, None))
    wp, wn = ws.get(need)
    rc = load().ffs_sample_lensemble(V.data_ptr(), lam.data_ptr(), L, K, dt, M, uniforms.data_ptr(),
                                     positions.data_ptr(), counts.data_ptr(), flags.data_ptr(), wp, wn,
                                     _stream_handle(stream, V.device))
    _check(rc)
    _keep_alive(stream, V, lam, uniforms, positions, counts, flags, ws.buf)
    return positions, counts, flags


def _positions_arg(positions: torch.Tensor):
    if not positions.is_cuda or positions.dtype != torch.int32 or positions.dim() != 2:
        raise FFSError("positions must be a CUDA int32 tensor [M][N']")
    return positions.contiguous()


def ffs_occupation(positions: torch.Tensor, L: int, stream=None) -> torch.Tensor:
    """occ[x] = number of samples with site x occupied (int64 [L]; uint64 counts in the library)."""
    positions = _positions_arg(positions)
    M, Np = positions.shape
    occ = torch.empty(L, dtype=torch.int64, device=positions.device)
    _check(load().ffs_occupation(positions.data_ptr(), M, Np, L, occ.data_ptr(),
                                 _stream_handle(stream, positions.device)))
    _keep_alive(stream, positions, occ)
    return occ


def ffs_pair_occupation(positions: torch.Tensor, W: int, stream=None) -> torch.Tensor:
    """pair[x][y] = number of samples with x and y occupied, x, y < W (int64 [W][W])."""
    positions = _positions_arg(positions)
    M, Np = positions.shape
    pair = torch.empty((W, W), dtype=torch.int64, device=positions.device)
    _check(load().ffs_pair_occupation(positions.data_ptr(), M, Np, W, pair.data_ptr(),
                                      _stream_handle(stream, positions.device)))
    _keep_alive(stream, positions, pair)
    return pair


def ffs_gutzwiller_reweight(positions: torch.Tensor, L: int, V: float, workspace: Optional[Workspace] = None,
                            stream=None):
    """Gutzwiller reweighting (Supp S5) of spinful samples (rows 2s up, 2s+1 down): returns
    result float64 [2 + L] = [<J^2>_0, <D>_J, <n_x>_J ...] and the D histogram int64 [N'+1]."""
    positions = _positions_arg(positions)
    M, Np = positions.shape
    if M % 2 or M == 0:
        raise FFSError("positions must hold an even, nonzero number of rows (up/down pairs)")
    res = torch.empty(2 + L, dtype=torch.float64, device=positions.device)
    dcount = torch.empty(Np + 1, dtype=torch.int64, device=positions.device)
    ws = workspace if workspace is not None else Workspace(positions.device)
    wp, wn = ws.get(int(load().ffs_gutzwiller_workspace_bytes(Np, L)))
    _check(load().ffs_gutzwiller_reweight(positions.data_ptr(), M // 2, Np, L, float(V), res.data_ptr(),
                                          dcount.data_ptr(), wp, wn, _stream_handle(stream, positions.device)))
    _keep_alive(stream, positions, res, dcount, ws.buf)
    return res, dcount


def ffs_sample_metropolis(U: torch.Tensor, uniforms: torch.Tensor, Nprime: int, Mcond: int,
                          workspace: Optional[Workspace] = None, stream=None):
    """Supp S7 variant: Mcond Metropolis updates per step (uniform discrete proposals).
    uniforms [M][N' + N'(1 + 2 Mcond)]; returns positions int32 [M][N'] and flags int32 [M]."""
    if not (U.is_cuda and uniforms.is_cuda) or U.dim() != 2:
        raise FFSError("U [L][N] and uniforms must be CUDA tensors")
    U = U.contiguous()
    uniforms = uniforms.contiguous()
    L, N = U.shape
    width = Nprime + Nprime * (1 + 2 * Mcond)
    if uniforms.dtype != torch.float64 or uniforms.dim() != 2 or uniforms.shape[1] != width:
        raise FFSError(f"uniforms must be float64 [M][{width}], got {tuple(uniforms.shape)}")
    M = uniforms.shape[0]
    dt = _dtype_code(U)
    positions = torch.empty((M, Nprime), dtype=torch.int32, device=U.device)
    flags = torch.empty(M, dtype=torch.int32, device=U.device)
    ws = workspace if workspace is not None else Workspace(U.device)
    need = int(load().ffs_metropolis_workspace_bytes(L, N, Nprime, Mcond, dt, M))
    if need == 0 and M > 0:
        _check(load().ffs_sample_metropolis(U.data_ptr(), L, N, dt, M, Nprime, Mcond, None, None, None, None, 0, None))
    wp, wn = ws.get(need)
    _check(load().ffs_sample_metropolis(U.data_ptr(), L, N, dt, M, Nprime, Mcond, uniforms.data_ptr(),
                                        positions.data_ptr(), flags.data_ptr(), wp, wn,
                                        _stream_handle(stream, U.device)))
    _keep_alive(stream, U, uniforms, positions, flags, ws.buf)
    return positions, flags


def ffs_sample_hkpv(U: torch.Tensor, uniforms: torch.Tensor, Nprime: Optional[int] = None,
                    workspace: Optional[Workspace] = None, stream=None):
    """Modified-HKPV comparator: uniforms [M][N'] selection draws;
    returns positions int32 [M][N'] and flags int32 [M]."""
    if not (U.is_cuda and uniforms.is_cuda) or U.dim() != 2:
        raise FFSError("U [L][N] and uniforms must be CUDA tensors")
    U = U.contiguous()
    uniforms = uniforms.contiguous()
    L, N = U.shape
    Np = uniforms.shape[1] if Nprime is None else Nprime
    if uniforms.dtype != torch.float64 or uniforms.dim() != 2 or uniforms.shape[1] != Np:
        raise FFSError(f"uniforms must be float64 [M][N'={Np}], got {tuple(uniforms.shape)}")
    M = uniforms.shape[0]
    dt = _dtype_code(U)
    positions = torch.empty((M, Np), dtype=torch.int32, device=U.device)
    flags = torch.empty(M, dtype=torch.int32, device=U.device)
    ws = workspace if workspace is not None else Workspace(U.device)
    need = int(load().ffs_hkpv_workspace_bytes(L, N, Np, dt, M))
    if need == 0 and M > 0:
        _check(load().ffs_sample_hkpv(U.data_ptr(), L, N, dt, M, Np, None, None, None, None, 0, None))
    wp, wn = ws.get(need)
    _check(load().ffs_sample_hkpv(U.data_ptr(), L, N, dt, M, Np, uniforms.data_ptr(), positions.data_ptr(),
                                  flags.data_ptr(), wp, wn, _stream_handle(stream, U.device)))
    _keep_alive(stream, U, uniforms, positions, flags, ws.buf)
    return positions, flags
