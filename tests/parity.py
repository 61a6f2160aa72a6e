"""Parity comparison between the CUDA path and the oracle (test infrastructure).

Positions: bit-exact, except at a CDF-boundary tie — at the first step where a sample's GPU and
oracle positions differ, the divergence is a tie iff the selection uniform lies within 1e-9 of
one of the oracle's normalised CDF values bracketing the oracle's choice (reading Q10). Tied
samples are counted and their later steps excluded; any other divergence is a failure.

Weights: normwise, max_x |w_gpu(x) - w_ref(x)| <= 1e-10 * max_x w_ref(x) per step, both
normalised to sum 1 (reading Q9).
"""
from __future__ import annotations

import numpy as np

from oracle import ref

TIE_EPS = 1e-9
WEIGHT_TOL = 1e-10


def compare_positions(U, uniforms, gpu_pos, ref_pos, Np):
    """Returns dict(n, exact, ties, failures=[(i, k, gpu, ref)])."""
    gpu_pos = np.asarray(gpu_pos)
    ref_pos = np.asarray(ref_pos)
    n = ref_pos.shape[0]
    diff = gpu_pos[:n] != ref_pos
    bad_rows = np.nonzero(diff.any(axis=1))[0]
    ties, failures = 0, []
    for i in bad_rows:
        k = int(np.argmax(diff[i]))
        _, w = ref.weights(U, uniforms[i:i + 1], Np=Np)
        F = np.cumsum(w[0, k])
        xs = int(ref_pos[i, k])
        u = uniforms[i, Np + k]
        lo = F[xs - 1] if xs > 0 else 0.0
        hi = F[xs]
        if abs(u - lo) < TIE_EPS or abs(u - hi) < TIE_EPS:
            ties += 1
        else:
            failures.append((int(i), k, int(gpu_pos[i, k]), xs, float(u), float(lo), float(hi)))
    return {"n": n, "exact": int(n - len(bad_rows)), "ties": ties, "failures": failures}


def compare_weights(gpu_w, ref_w, gpu_pos, ref_pos):
    """Normwise relative error per (sample, step) along the common path prefix; returns max."""
    worst = 0.0
    S, Np, _ = ref_w.shape
    for i in range(S):
        for k in range(Np):
            a, b = gpu_w[i, k], ref_w[i, k]
            err = np.max(np.abs(a - b)) / max(np.max(b), 1e-300)
            worst = max(worst, err)
            if gpu_pos[i, k] != ref_pos[i, k]:
                break  # paths diverge after this step (tie); later weights are not comparable
    return worst
