"""Seeded synthetic inputs for the FFS hot path: orbital matrices U and Philox uniforms.

This module is shared by the CUDA path's tests/bench AND by the oracle's tests. It holds
NO arithmetic of the sampling method itself (no elimination, no weights, no selection):
only the construction of the one-body problems whose N lowest orbitals form U (setup,
never timed), and the counter-based uniforms the method consumes.

Recipes follow BASELINE.json `configs` and SURVEY.md §8(d) (readings Q14/Q15 in DESIGN.md):

* C1 tiny     : U = Q of reduced QR of a seeded 16x4 N(0,1) matrix.
* C2 dw       : open chain L=256, t=1, V(x)=4((x-128)^2/64^2-1)^2; N=32 lowest.
* C3 anderson : open chain L=1024, t=1, eps_x ~ U[-2,2] (seed 0); N=128 lowest; marginal N'=16.
* C4 peierls  : 64x64 torus, site 64*x+y, Landau gauge (x-bonds -1, y-bonds -exp(i 2 pi phi x)),
                phi=1/16, + U[-1,1] disorder; complex128; N=512 lowest.
* C5 dpp      : B = diag(q) G, G ~ N(0,1)^{16384x1024}, q = exp(0.5 z), z ~ N(0,1) (G drawn first);
                U = Q of reduced QR (projection DPP with every eigenvector of C = B B^T kept,
                PAPER.md:178-180); N=1024; marginal N'=64.

Uniform rows (reading Q6/Q7): uniforms[i, 0:N'] drive the permutation draw,
uniforms[i, N':2N'] drive the N' inverse-CDF selections.
"""
from __future__ import annotations

import dataclasses
import hashlib
import os
from typing import Optional

import numpy as np

F64 = 0
C128 = 1


@dataclasses.dataclass(frozen=True)
class Config:
    name: str
    L: int
    N: int
    M: int
    Nprime: int           # steps per sample (== N for full sampling)
    dtype: int            # F64 or C128
    index: int            # BASELINE.json configs[] index (uniform seed = 1000 + index)
    recipe: str           # which U builder
    marginal_M: Optional[int] = None  # extra marginal workload (BASELINE.json) if any
    marginal_Np: Optional[int] = None

    @property
    def uniform_seed(self) -> int:
        return 1000 + self.index


CONFIGS = {
    "tiny": Config("tiny", 16, 4, 200000, 4, F64, 0, "qr_gauss"),
    "dw": Config("dw", 256, 32, 65536, 32, F64, 1, "double_well"),
    "anderson": Config("anderson", 1024, 128, 16384, 128, F64, 2, "anderson",
                       marginal_M=16384, marginal_Np=16),
    "peierls": Config("peierls", 4096, 512, 4096, 512, C128, 3, "peierls"),
    "dpp": Config("dpp", 16384, 1024, 1024, 1024, F64, 4, "dpp",
                  marginal_M=8192, marginal_Np=64),
}


def lowest_orbitals(H: np.ndarray, N: int) -> np.ndarray:
    """N lowest eigenvectors of a Hermitian one-body Hamiltonian (setup, not timed)."""
    w, v = np.linalg.eigh(H)
    return np.ascontiguousarray(v[:, :N])


def chain_hamiltonian(onsite: np.ndarray, t: float = 1.0) -> np.ndarray:
    """Open-boundary nearest-neighbour chain: H = -t sum (c+_x c_{x+1} + h.c.) + sum v_x n_x."""
    L = onsite.shape[0]
    H = np.diag(onsite.astype(np.float64))
    idx = np.arange(L - 1)
    H[idx, idx + 1] = -t
    H[idx + 1, idx] = -t
    return H


def build_u_qr_gauss(L: int, N: int, seed: int = 0) -> np.ndarray:
    G = np.random.default_rng(seed).standard_normal((L, N))
    Q, _ = np.linalg.qr(G)
    return np.ascontiguousarray(Q)


def build_u_double_well(L: int = 256, N: int = 32) -> np.ndarray:
    x = np.arange(L, dtype=np.float64)
    V = 4.0 * ((x - L / 2) ** 2 / (L / 4) ** 2 - 1.0) ** 2
    return lowest_orbitals(chain_hamiltonian(V), N)


def build_u_anderson(L: int = 1024, N: int = 128, W: float = 2.0, seed: int = 0) -> np.ndarray:
    eps = np.random.default_rng(seed).uniform(-W, W, L)
    return lowest_orbitals(chain_hamiltonian(eps), N)


def build_u_peierls(Lx: int = 64, Ly: int = 64, N: int = 512, phi: float = 1.0 / 16,
                    W: float = 1.0, seed: int = 0) -> np.ndarray:
    L = Lx * Ly
    H = np.zeros((L, L), dtype=np.complex128)
    site = lambda x, y: (x % Lx) * Ly + (y % Ly)
    for x in range(Lx):
        for y in range(Ly):
            s = site(x, y)
            sx = site(x + 1, y)
            H[s, sx] += -1.0
            H[sx, s] += -1.0
            sy = site(x, y + 1)
            ph = np.exp(2j * np.pi * phi * x)
            H[s, sy] += -ph
            H[sy, s] += -np.conj(ph)
    eps = np.random.default_rng(seed).uniform(-W, W, L)
    H[np.arange(L), np.arange(L)] += eps
    return lowest_orbitals(H, N)


def build_u_dpp(L: int = 16384, N: int = 1024, seed: int = 0) -> np.ndarray:
    rng = np.random.default_rng(seed)
    G = rng.standard_normal((L, N))
    q = np.exp(0.5 * rng.standard_normal(L))
    Q, _ = np.linalg.qr(q[:, None] * G)
    return np.ascontiguousarray(Q)


def random_orthonormal(L: int, N: int, seed: int, complex_: bool = False) -> np.ndarray:
    """Random L x N matrix with orthonormal columns (Fig. 3B-style inputs; small test cases)."""
    rng = np.random.default_rng(seed)
    G = rng.standard_normal((L, N))
    if complex_:
        G = G + 1j * rng.standard_normal((L, N))
    Q, _ = np.linalg.qr(G)
    return np.ascontiguousarray(Q)


# Outside the repo so the (up to 128 MB) matrices never travel with a gpurun snapshot.
_CACHE_DIR = os.environ.get("FFS_INPUT_CACHE", "/tmp/ffs_input_cache")


def build_u(cfg: Config) -> np.ndarray:
    """U for a registered config; cached on disk (git-ignored) because C4's eigh takes ~1 min."""
    # keyed by the config AND this file's recipe source, so an edited generator never serves a
    # stale matrix
    key = hashlib.sha256((repr(cfg) + open(__file__).read()).encode()).hexdigest()[:16]
    path = os.path.join(_CACHE_DIR, f"U_{cfg.name}_{key}.npy")
    if os.path.exists(path):
        try:
            return np.load(path)
        except Exception:
            pass
    if cfg.recipe == "qr_gauss":
        U = build_u_qr_gauss(cfg.L, cfg.N, 0)
    elif cfg.recipe == "double_well":
        U = build_u_double_well(cfg.L, cfg.N)
    elif cfg.recipe == "anderson":
        U = build_u_anderson(cfg.L, cfg.N)
    elif cfg.recipe == "peierls":
        U = build_u_peierls(64, 64, cfg.N)
    elif cfg.recipe == "dpp":
        U = build_u_dpp(cfg.L, cfg.N)
    else:
        raise ValueError(cfg.recipe)
    try:
        os.makedirs(_CACHE_DIR, exist_ok=True)
        tmp = path + f".tmp{os.getpid()}"
        np.save(tmp, U)
        os.replace(tmp + ".npy" if not tmp.endswith(".npy") else tmp, path)
    except OSError:
        pass
    return U


# ---------------------------------------------------------------- L-ensemble workload
@dataclasses.dataclass(frozen=True)
class LensConfig:
    """A DPP-summarisation-shaped L-ensemble: L items with D-dimensional features B = diag(q) G,
    G ~ N(0,1)^{L x D} (seed), quality q = exp(0.5 z), z ~ N(0,1) (the C5 recipe at L = 1024, the
    paper's Fig. 3B chain length); C = s B B^T with the scale s chosen so that the expected sample
    size sum_j lambda_j/(lambda_j+1) equals n_mean (the paper's summaries keep a few sentences per
    article; here a larger n_mean so every sample runs tens of FFS steps). Eigenvectors / values
    come from the SVD of B (setup, not timed)."""
    name: str = "lens"
    L: int = 1024
    D: int = 256
    n_mean: float = 64.0
    M: int = 16384
    seed: int = 0

    @property
    def uniform_seed(self) -> int:
        return 1005


LENS = LensConfig()


def build_lensemble(cfg: LensConfig = LENS, L: Optional[int] = None, D: Optional[int] = None,
                    n_mean: Optional[float] = None, seed: Optional[int] = None, complex_: bool = False):
    """(V [L][D], lam [D]) of the L-ensemble kernel C = V diag(lam) V^dagger."""
    L = cfg.L if L is None else L
    D = cfg.D if D is None else D
    n_mean = cfg.n_mean if n_mean is None else n_mean
    rng = np.random.default_rng(cfg.seed if seed is None else seed)
    G = rng.standard_normal((L, D))
    if complex_:
        G = G + 1j * rng.standard_normal((L, D))
    q = np.exp(0.5 * rng.standard_normal(L))
    V, sig, _ = np.linalg.svd(q[:, None] * G, full_matrices=False)
    s2 = sig ** 2
    lo, hi = -60.0, 60.0  # bisection on log s: expected size sum s s2/(1 + s s2) = n_mean
    for _ in range(200):
        mid = 0.5 * (lo + hi)
        e = np.sum(np.exp(mid) * s2 / (1.0 + np.exp(mid) * s2))
        lo, hi = (mid, hi) if e < n_mean else (lo, mid)
    lam = np.exp(0.5 * (lo + hi)) * s2
    return np.ascontiguousarray(V), np.ascontiguousarray(lam)


def lens_uniforms(M: int, K: int, seed: int) -> np.ndarray:
    """[M][3K] fp64 uniforms (keep draws | permutation draws | selections), numpy Philox."""
    return np.random.Generator(np.random.Philox(seed)).random((M, 3 * K))


# ---------------------------------------------------------------- Supp S7 workload (continuous models)
@dataclasses.dataclass(frozen=True)
class MetroConfig:
    """Continuous-model stand-in for the Supp S7 variant: N fermions in a box,
    discretised on a fine grid of L sites (the "large number of lattice sites L" that makes the
    explicit sampler inefficient); U = the N lowest box orbitals
    U[x, n] = sqrt(2/(L+1)) sin(pi (n+1)(x+1)/(L+1)) (exact eigenvectors of the open chain, so
    orthonormal without a factorisation). M_cond updates per step, N' = N."""
    name: str = "metro"
    L: int = 1 << 20
    N: int = 64
    Mc: int = 32
    M: int = 16384

    @property
    def uniform_seed(self) -> int:
        return 1006


METRO = MetroConfig()


def build_box_orbitals(L: int, N: int) -> np.ndarray:
    x = np.arange(1, L + 1, dtype=np.float64)[:, None]
    n = np.arange(1, N + 1, dtype=np.float64)[None, :]
    return np.ascontiguousarray(np.sqrt(2.0 / (L + 1)) * np.sin(np.pi * n * x / (L + 1)))


def metro_uniforms(M: int, Np: int, Mc: int, seed: int) -> np.ndarray:
    """[M][N' + N'(1 + 2 Mc)] fp64 uniforms: permutation draws, then per step u_init and
    (u_prop, u_acc) x Mc (numpy Philox)."""
    return np.random.Generator(np.random.Philox(seed)).random((M, Np + Np * (1 + 2 * Mc)))


def u_sha256(U: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(U).tobytes()).hexdigest()


def workload_uniforms(cfg: Config, marginal: bool = False) -> np.ndarray:
    """Uniforms of a registered workload: seed 1000+index (full) or 1100+index (marginal)."""
    if marginal:
        return uniforms(cfg.marginal_M, cfg.marginal_Np, cfg.uniform_seed + 100)
    return uniforms(cfg.M, cfg.Nprime, cfg.uniform_seed)


def uniforms(M: int, Nprime: int, seed: int) -> np.ndarray:
    """[M][2N'] fp64 uniforms in [0,1) from numpy's counter-based Philox generator."""
    return np.random.Generator(np.random.Philox(seed)).random((M, 2 * Nprime))


def u_as_f64_view(U: np.ndarray) -> np.ndarray:
    """Interleaved (re,im) float64 view for complex U (ABI dtype C128); real U unchanged."""
    U = np.ascontiguousarray(U)
    if np.iscomplexobj(U):
        return U.view(np.float64).reshape(U.shape[0], U.shape[1] * 2)
    return U.astype(np.float64, copy=False)


def dtype_of(U: np.ndarray) -> int:
    return C128 if np.iscomplexobj(U) else F64
