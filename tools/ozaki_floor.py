"""How many int8 slices would an Ozaki-style emulation of the dense-path GEMM P = U Y need for
the weights to stay within the 1e-10 normwise bound? (CPU, numpy; development)

For one sample of a config, the positions of its first k0 draws come from the oracle; then
W = A^{-1} V[X, k0:k0+B] and the panel P = V[:, k0:k0+B] - V[:, 0:k0] W = U Y (Y scattered as in
ffs_dense.cuh). The emulation scales each row of U and each column of Y by a power of two,
splits the scaled values into s signed 7-bit slices, multiplies slice pairs (i + j < s) exactly
(integer-valued fp64 matmuls) and sums. Reported: max_x |w_emul(x) - w(x)| / max_x w(x) of the
normalised weights of the block's first column.
    python tools/ozaki_floor.py [config] [k0 ...]"""
import sys
import numpy as np
from oracle import ref
from paper_2109_07358_b200 import inputs


def split(M, axis, s):
    """M ~= sum_i S_i * 2^(-7(i+1)) * scale (scale per row (axis=1) or column (axis=0))"""
    mx = np.max(np.abs(M), axis=axis, keepdims=True)
    e = np.ceil(np.log2(np.where(mx > 0, mx, 1.0)))
    R = M / 2.0 ** e  # |R| <= 1
    out = []
    for i in range(s):
        q = np.trunc(R * 2.0 ** 7)
        out.append(q)
        R = R * 2.0 ** 7 - q
    return out, e


def emul(U, Y, s):
    As, ea = split(U, 1, s)
    Bs, eb = split(Y, 0, s)
    P = np.zeros((U.shape[0], Y.shape[1]))
    for i in range(s):
        for j in range(s - i):
            P += (As[i] @ Bs[j]) * 2.0 ** (-7 * (i + 1) - 7 * (j + 1))
    return P * 2.0 ** ea * 2.0 ** eb


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "dpp"
    cfg = inputs.CONFIGS[name]
    U = inputs.build_u(cfg)
    N, L, B = cfg.N, cfg.L, 8
    ks = [int(a) for a in sys.argv[2:]] or [N // 4, N // 2, 3 * N // 4, N - 2 * B]
    uni = inputs.uniforms(1, N, cfg.uniform_seed)
    pos = ref.sample(U, uni)[0]
    # permutation (reading Q6)
    m = list(range(N))
    for j in range(N):
        n = N - j
        r = j + min(n - 1, int(np.floor(uni[0, j] * n)))
        m[j], m[r] = m[r], m[j]
    m = np.array(m)
    for k0 in ks:
        X = pos[:k0]
        V = U[:, m]
        A = V[X, :k0]
        W = np.linalg.solve(A, V[X, k0:k0 + B]) if k0 else np.zeros((0, B))
        Y = np.zeros((N, B), dtype=U.dtype)
        Y[m[:k0]] = -W
        Y[m[k0:k0 + B], np.arange(B)] = 1.0
        P = U @ Y
        w = np.abs(P[:, 0]) ** 2
        w[X] = 0
        w /= w.sum()
        row = [f"k0={k0:5d} |W|max={np.abs(W).max() if k0 else 0:9.3g}"]
        for s in (4, 5, 6, 7, 8):
            if np.iscomplexobj(U):
                Ur, Ui, Yr, Yi = U.real, U.imag, Y.real, Y.imag
                Pe = (emul(Ur, Yr, s) - emul(Ui, Yi, s)) + 1j * (emul(Ur, Yi, s) + emul(Ui, Yr, s))
            else:
                Pe = emul(U, Y, s)
            we = np.abs(Pe[:, 0]) ** 2
            we[X] = 0
            we /= we.sum()
            row.append(f"s={s}: {np.max(np.abs(we - w)) / w.max():8.2e}")
        print(name, "  ".join(row), flush=True)


if __name__ == "__main__":
    main()
