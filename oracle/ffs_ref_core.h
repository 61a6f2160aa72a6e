/* ORACLE CORE — TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).
 *
 * One FFS sample, written step by step in the paper's order and notation.
 * This file is #included twice by ffs_ref.c: once with SCALAR = double (real U, dtype F64)
 * and once with SCALAR = double _Complex (complex U, dtype C128). The macros
 *   SCALAR, ABS2(z) = |z|^2, SFX(name) = name-suffix
 * are defined by the includer. Nothing here is shared with the CUDA path.
 *
 * Notation (Supp S1 PAPER.md:242-256):
 *   U       : L x N, orthonormal columns, row-major, U[x*N + c]
 *   m       : random permutation of (0..N-1); only m[0..Np) is used
 *   u_x     : the k-dimensional row vector U_{x,(m_1..m_k)}
 *   R       : the iteratively Gauss-eliminated rows of u_{x_1..x_{k-1}}, kept in the permuted
 *             column order over ncols columns ("always carry out Gaussian elimination in the full
 *             N-dimensional space"; ncols = Np, reading Q11 in DESIGN.md)
 *   h       : k-dim unit normal vector, perpendicular to u_{x_1..x_{k-1}} (Eq. 3)
 *   w(x)    : |u_x^T h|^2  (Eq. 3; bilinear u^T h, no conjugation: reading Q3)
 */

/* Unit normal vector h of step k (1-based) from the k-1 reduced rows R (PAPER.md:255:
 * "the normal vector h can be determined with another k(k-1)/2 additions and summations"):
 * back-substitution of R[0:k-1, 0:k] h = 0 with the free component h[k-1] = 1, then normalise.
 * Returns |h'|^2 of the un-normalised h' (h'[k-1] = 1) through *hnorm2. */
static void SFX(normal_vector)(const SCALAR* R, int64_t ncols, int64_t k, SCALAR* h, double* hnorm2)
{
    h[k - 1] = 1.0;
    for (int64_t i = k - 2; i >= 0; --i) {
        SCALAR acc = 0.0;
        for (int64_t j = i + 1; j <= k - 1; ++j) acc += R[i * ncols + j] * h[j];
        h[i] = -acc / R[i * ncols + i];
    }
    double n2 = 0.0;
    for (int64_t j = 0; j < k; ++j) n2 += ABS2(h[j]);
    *hnorm2 = n2;
    double inv = 1.0 / sqrt(n2);
    for (int64_t j = 0; j < k; ++j) h[j] *= inv;
}

/* advance_elimination: append the row u_{x_{k-1}} (all ncols permuted columns)
 * as R[k-2], eliminating its first k-2 entries against the k-2 rows already stored. */
static void SFX(advance_elimination)(const SCALAR* U, int64_t N, const int32_t* m, int64_t x,
                                     SCALAR* R, int64_t ncols, int64_t k)
{
    SCALAR* row = R + (k - 2) * ncols;
    for (int64_t j = 0; j < ncols; ++j) row[j] = U[x * N + m[j]];
    for (int64_t i = 0; i <= k - 3; ++i) {
        SCALAR f = row[i] / R[i * ncols + i];
        row[i] = 0.0;
        for (int64_t j = i + 1; j < ncols; ++j) row[j] -= f * R[i * ncols + j];
    }
}

/* One sample of Np sequential steps ("the fermion position x_k is drawn
 * according to the conditional probability distribution, with the index k iteratively increased
 * from 1 to N step by step"; marginal N_< = Np < N stops the loop early).
 *
 *   m        : permutation (already drawn), length >= Np
 *   u_sel    : Np selection uniforms in [0,1)
 *   forced   : if non-NULL, teacher forcing: x_k := forced[k-1] (weights still computed)
 *   x_out    : Np positions (0-based, sampling order)
 *   w_trace  : if non-NULL, [Np][L] normalised conditional weights w/T
 *   hn2_out  : if non-NULL, [Np] |h'|^2 (un-normalised normal vector with h'[k-1]=1)
 *   tot_out  : if non-NULL, [Np] T = sum_x w(x) with unit h
 *   scratch  : R (Np*Np SCALAR) + h (Np SCALAR) + w (L double) + chosen (L char) — caller-provided
 * Returns flags: bit0 = a step had a non-finite or non-positive total T,
 *                bit1 = a selected normalised weight was < 1e-12.                            */
static int SFX(sample_chain)(const SCALAR* U, int64_t L, int64_t N, int64_t Np, const int32_t* m,
                             const double* u_sel, const int32_t* forced, int32_t* x_out,
                             double* w_trace, double* hn2_out, double* tot_out,
                             SCALAR* R, SCALAR* h, double* w, char* chosen)
{
    const int64_t ncols = Np;
    int flags = 0;
    memset(chosen, 0, (size_t)L);
    for (int64_t k = 1; k <= Np; ++k) {
        if (k >= 2) SFX(advance_elimination)(U, N, m, x_out[k - 2], R, ncols, k);
        double hn2;
        SFX(normal_vector)(R, ncols, k, h, &hn2);
        /* conditional weights for all L candidates ("Calculating the inner product
         * u_{x_k}^T h for all x_k"); already-chosen sites forced to 0 (reading Q5/SPEC.md:211) */
        double T = 0.0;
        for (int64_t x = 0; x < L; ++x) {
            double wx = 0.0;
            if (!chosen[x]) {
                SCALAR s = 0.0;
                for (int64_t j = 0; j < k; ++j) s += U[x * N + m[j]] * h[j];
                wx = ABS2(s);
            }
            w[x] = wx;
            T += wx;
        }
        /* inverse-CDF draw (reading Q4/Q5): x_k = min{x : C(x) > u*T}, C the inclusive prefix
         * sum in index order; if none, the largest x with w(x) > 0. */
        int64_t sel = -1;
        if (!(T > 0.0) || !isfinite(T)) {
            flags |= 1;
            for (int64_t x = 0; x < L; ++x) if (!chosen[x]) { sel = x; break; }
        } else if (!forced) {
            double t = u_sel[k - 1] * T, C = 0.0;
            for (int64_t x = 0; x < L; ++x) {
                C += w[x];
                if (C > t) { sel = x; break; }
            }
            if (sel < 0)
                for (int64_t x = L - 1; x >= 0; --x) if (w[x] > 0.0) { sel = x; break; }
        }
        if (forced) sel = forced[k - 1];
        if (sel < 0) sel = 0; /* unreachable for L >= N: some unchosen site always exists */
        if (T > 0.0 && w[sel] / T < 1e-12) flags |= 2;
        x_out[k - 1] = (int32_t)sel;
        chosen[sel] = 1;
        if (w_trace)
            for (int64_t x = 0; x < L; ++x) w_trace[(k - 1) * L + x] = (T > 0.0) ? w[x] / T : 0.0;
        if (hn2_out) hn2_out[k - 1] = hn2;
        if (tot_out) tot_out[k - 1] = T;
    }
    return flags;
}

/* Continuous / large-L variant (Supp S7): the same permutation, elimination and
 * normal vector h as sample_chain, but x_k is drawn by a Metropolis chain of Mc updates instead of
 * the explicit inverse-CDF draw over all L candidates: "A trial random ... update is proposed
 * (x_k -> x_k + dx), and then accepted with probability |u_{x_k+dx}^T h|^2 / |u_{x_k}^T h|^2"
 * (PAPER.md:385-386); "The update is iterated for M_cond times"; for problems with
 * large L "replace the continuous update x_k -> x_k + dx by a discrete update x_k -> x_k'"
 * (PAPER.md:393). Readings (Q16-Q18): the chain starts at x = floor(u_init L); the
 * discrete update proposes x' = floor(u_prop L) (uniform over the sites: a symmetric proposal);
 * the move is accepted iff u_acc * w(x) < w(x') (= u_acc < min(1, w(x')/w(x)), and a zero-weight
 * start moves to the first positive-weight proposal); chosen sites have w = 0 (Pauli exclusion).
 *   u       : [Np perm draws | Np x (1 + 2 Mc) chain draws: init, (prop, acc) x Mc]
 *   margin  : if non-NULL, [Np] the smallest |u_acc - w(x')/w(x)| over the step's decisions with
 *             w(x) > 0 (how close a decision came to flipping; tie detection in the parity tests)
 * Returns flags: bit0 = some h had a non-finite norm, bit2 = a chain ended on a zero-weight site. */
static int SFX(sample_metropolis)(const SCALAR* U, int64_t L, int64_t N, int64_t Np, int64_t Mc, const int32_t* m,
                                  const double* u, int32_t* x_out, double* margin, SCALAR* R, SCALAR* h, char* chosen)
{
    const int64_t ncols = Np;
    int flags = 0;
    memset(chosen, 0, (size_t)L);
    for (int64_t k = 1; k <= Np; ++k) {
        if (k >= 2) SFX(advance_elimination)(U, N, m, x_out[k - 2], R, ncols, k);
        double hn2;
        SFX(normal_vector)(R, ncols, k, h, &hn2);
        if (!isfinite(hn2)) flags |= 1;
        const double* uc = u + Np + (k - 1) * (1 + 2 * Mc);
        double mg = INFINITY;
        int64_t x = (int64_t)floor(uc[0] * (double)L);
        if (x > L - 1) x = L - 1;
        double wx = 0.0;
        if (!chosen[x]) {
            SCALAR s = 0.0;
            for (int64_t j = 0; j < k; ++j) s += U[x * N + m[j]] * h[j];
            wx = ABS2(s);
        }
        for (int64_t t = 0; t < Mc; ++t) {
            int64_t xp = (int64_t)floor(uc[1 + 2 * t] * (double)L);
            if (xp > L - 1) xp = L - 1;
            double wp = 0.0;
            if (!chosen[xp]) {
                SCALAR s = 0.0;
                for (int64_t j = 0; j < k; ++j) s += U[xp * N + m[j]] * h[j];
                wp = ABS2(s);
            }
            const double ua = uc[2 + 2 * t];
            if (wx > 0.0 && fabs(ua - wp / wx) < mg) mg = fabs(ua - wp / wx);
            if (ua * wx < wp) {
                x = xp;
                wx = wp;
            }
        }
        if (!(wx > 0.0)) flags |= 4;
        x_out[k - 1] = (int32_t)x;
        chosen[x] = 1;
        if (margin) margin[k - 1] = mg;
    }
    return flags;
}

/* Modified HKPV sampler (the paper's comparison method: "improved from O(N^3 L) to
 * O(N^2 L) with certain modification", "the modified HPKV algorithm requires 2LN^2
 * operations"; its steps as SPEC.md:238-246 states them): the chain rule on the projection kernel
 * K = U U^dagger without forming K. r_1(x) = |u_x|^2; at step k, x_k ~ r_k (inverse CDF with the
 * selection rule of reading Q5; chosen sites 0, rounding residues below 0 clamped to 0); then
 * e_k = u_{x_k} orthonormalised against e_1..e_{k-1} (modified Gram-Schmidt, Hermitian inner
 * product <a, b> = sum_n a_n conj(b_n)) and r_{k+1}(x) = r_k(x) - |<u_x, e_k>|^2 for every x
 * (L N multiply-adds per step: 2 L N^2 operations in total).
 *   u_sel : Np selection uniforms;  w_trace / tot_out as sample_chain (normalised r_k, and T_k)
 *   E     : scratch Np x N SCALAR, r : scratch L doubles */
static int SFX(hkpv_chain)(const SCALAR* U, int64_t L, int64_t N, int64_t Np, const double* u_sel, int32_t* x_out,
                           double* w_trace, double* tot_out, SCALAR* E, double* r, char* chosen)
{
    int flags = 0;
    memset(chosen, 0, (size_t)L);
    for (int64_t x = 0; x < L; ++x) {
        double a = 0.0;
        for (int64_t n = 0; n < N; ++n) a += ABS2(U[x * N + n]);
        r[x] = a;
    }
    for (int64_t k = 1; k <= Np; ++k) {
        double T = 0.0;
        for (int64_t x = 0; x < L; ++x) {
            double wx = (chosen[x] || !(r[x] > 0.0)) ? 0.0 : r[x];
            T += wx;
        }
        int64_t sel = -1;
        if (!(T > 0.0) || !isfinite(T)) {
            flags |= 1;
            for (int64_t x = 0; x < L; ++x) if (!chosen[x]) { sel = x; break; }
        } else {
            double t = u_sel[k - 1] * T, C = 0.0;
            for (int64_t x = 0; x < L; ++x) {
                double wx = (chosen[x] || !(r[x] > 0.0)) ? 0.0 : r[x];
                C += wx;
                if (wx > 0.0 && C > t) { sel = x; break; }
            }
            if (sel < 0)
                for (int64_t x = L - 1; x >= 0; --x)
                    if (!chosen[x] && r[x] > 0.0) { sel = x; break; }
        }
        if (sel < 0) sel = 0;
        if (w_trace)
            for (int64_t x = 0; x < L; ++x)
                w_trace[(k - 1) * L + x] = (T > 0.0 && !chosen[x] && r[x] > 0.0) ? r[x] / T : 0.0;
        if (tot_out) tot_out[k - 1] = T;
        if (T > 0.0 && r[sel] / T < 1e-12) flags |= 2;
        x_out[k - 1] = (int32_t)sel;
        chosen[sel] = 1;
        if (k == Np) break;
        /* e_k: modified Gram-Schmidt of u_{x_k} against e_1..e_{k-1} */
        SCALAR* e = E + (k - 1) * N;
        for (int64_t n = 0; n < N; ++n) e[n] = U[sel * N + n];
        for (int64_t j = 0; j < k - 1; ++j) {
            const SCALAR* ej = E + j * N;
            SCALAR c = 0.0;
            for (int64_t n = 0; n < N; ++n) c += e[n] * CONJ(ej[n]);
            for (int64_t n = 0; n < N; ++n) e[n] -= c * ej[n];
        }
        double nrm = 0.0;
        for (int64_t n = 0; n < N; ++n) nrm += ABS2(e[n]);
        nrm = sqrt(nrm);
        for (int64_t n = 0; n < N; ++n) e[n] /= nrm;
        /* residual update for every candidate */
        for (int64_t x = 0; x < L; ++x) {
            SCALAR c = 0.0;
            for (int64_t n = 0; n < N; ++n) c += U[x * N + n] * CONJ(e[n]);
            r[x] -= ABS2(c);
        }
    }
    return flags;
}
