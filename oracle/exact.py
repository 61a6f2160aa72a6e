"""ORACLE PINS — TEST INFRASTRUCTURE ONLY.

Plain definitions from PAPER.md, written with library primitives (numpy det / SVD /
itertools), used by tests/test_oracle.py to pin the C oracle to something other than itself.
Nothing here is used by the CUDA path.
"""
from __future__ import annotations

import itertools
import math

import numpy as np


def set_probabilities(U: np.ndarray):
    """Eq. 1 summed over the N! orderings of a set S: P(S) = |det U_{S,n}|^2.
    Returns (list of sorted index tuples, probabilities)."""
    L, N = U.shape
    subsets = list(itertools.combinations(range(L), N))
    p = np.array([abs(np.linalg.det(U[list(S), :])) ** 2 for S in subsets])
    return subsets, p


def ordered_probability(U: np.ndarray, x) -> float:
    """Eq. 1 for an ordered configuration x: |det U_{x,n}|^2 / N!."""
    N = U.shape[1]
    return abs(np.linalg.det(U[list(x), :])) ** 2 / math.factorial(N)


def det_conditional(U: np.ndarray, m, prefix) -> np.ndarray:
    """Conditional of Eq. 2 as a determinant ratio, normalised over x (reading Q1):
    P(x | prefix; m) = |det U_{(prefix,x),(m_1..m_k)}|^2 / sum_y |det U_{(prefix,y),(m_1..m_k)}|^2."""
    L = U.shape[0]
    k = len(prefix) + 1
    cols = list(m[:k])
    d = np.zeros(L)
    for x in range(L):
        if x in prefix:
            continue
        d[x] = abs(np.linalg.det(U[np.ix_(list(prefix) + [x], cols)])) ** 2
    return d / d.sum()


def nullvec_conditional(U: np.ndarray, m, prefix) -> np.ndarray:
    """Eq. 3 by definition: h = unit vector with u_{x_j}^T h = 0 for j < k (the
    bilinear null space of B = U_{prefix,(m_1..m_k)}, taken from the SVD), w(x) = |u_x^T h|^2."""
    L = U.shape[0]
    k = len(prefix) + 1
    cols = list(m[:k])
    if k == 1:
        h = np.ones(1, dtype=U.dtype)
    else:
        B = U[np.ix_(list(prefix), cols)]
        _, _, Vh = np.linalg.svd(B)
        h = np.conj(Vh[-1, :])          # B @ conj(Vh[-1]) = 0 (last right singular vector)
    w = np.abs(U[:, cols] @ h) ** 2
    w[list(prefix)] = 0.0
    return w / w.sum()


def ordered_marginal_probability(U: np.ndarray, xs) -> float:
    """Ordered N'-point marginal of Eq. 1: for a projection kernel K = U U^dagger,
    P(x_1..x_{N'}) = det[K(x_a, x_b)] (N-N')!/N!  (correlation-function identity)."""
    N = U.shape[1]
    K = U @ U.conj().T
    Np = len(xs)
    sub = K[np.ix_(list(xs), list(xs))]
    return float(np.real(np.linalg.det(sub))) * math.factorial(N - Np) / math.factorial(N)


def pooled_chisquare(observed: np.ndarray, expected: np.ndarray, min_expected: float = 5.0):
    """Chi-square with ascending-expectation pooling until every bin has E >= min_expected
    (SURVEY.md §8c). Returns (statistic, dof, p_value, n_bins)."""
    from scipy import stats

    order = np.argsort(expected)
    o = observed[order].astype(np.float64)
    e = expected[order].astype(np.float64)
    bins_o, bins_e = [], []
    co = ce = 0.0
    for oi, ei in zip(o, e):
        co += oi
        ce += ei
        if ce >= min_expected:
            bins_o.append(co)
            bins_e.append(ce)
            co = ce = 0.0
    if ce > 0:
        if bins_e:
            bins_o[-1] += co
            bins_e[-1] += ce
        else:
            bins_o.append(co)
            bins_e.append(ce)
    bo, be = np.array(bins_o), np.array(bins_e)
    stat = float(((bo - be) ** 2 / be).sum())
    dof = len(bo) - 1
    return stat, dof, float(stats.chi2.sf(stat, dof)), len(bo)


def lensemble_set_probabilities(V: np.ndarray, lam: np.ndarray):
    """L-ensemble law of the DPP pipeline by its definition: with the kernel
    C = V diag(lam) V^dagger, P(S) = det(C_S) / det(I + C) for every subset S of the L items
    (the empty set has det(C_empty) = 1). Returns (list of sorted index tuples, probabilities)."""
    L = V.shape[0]
    C = (V * lam[None, :]) @ V.conj().T
    Z = float(np.real(np.linalg.det(np.eye(L) + C)))
    subsets, p = [], []
    for n in range(L + 1):
        for S in itertools.combinations(range(L), n):
            subsets.append(S)
            p.append(1.0 if n == 0 else float(np.real(np.linalg.det(C[np.ix_(S, S)]))))
    return subsets, np.array(p) / Z


def gutzwiller_exact(U: np.ndarray, V: float):
    """Exact Gutzwiller-projected expectations by enumeration (Supp S5): every
    spinful configuration (S_up, S_dn) of the free ensemble has P_0 = P(S_up) P(S_dn) with
    P(S) = |det U_S|^2 (Eq. 1); the interacting distribution is P_J ∝ J^2 P_0, J^2 = exp(-V D),
    D = |S_up ∩ S_dn| (Eq. 4). Returns dict with <J^2>_0, <D>_J, <n_x>_J, and the per-configuration
    arrays (p0, J2, D, n) for error estimates."""
    subsets, p = set_probabilities(U)
    L = U.shape[0]
    p0, J2, D, n = [], [], [], []
    for a, pa in zip(subsets, p):
        for b, pb in zip(subsets, p):
            d = len(set(a) & set(b))
            occ = np.zeros(L)
            occ[list(a)] += 1
            occ[list(b)] += 1
            p0.append(pa * pb)
            J2.append(np.exp(-V * d))
            D.append(d)
            n.append(occ)
    p0, J2, D, n = map(np.array, (p0, J2, D, n))
    Z = np.sum(p0 * J2)
    return {"J2_0": Z, "D_J": np.sum(p0 * J2 * D) / Z, "n_J": (p0 * J2) @ n / Z,
            "p0": p0, "J2": J2, "D": D, "n": n}
