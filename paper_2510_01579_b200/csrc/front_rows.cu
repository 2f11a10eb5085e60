// Register-resident FP64 front-end for n_t <= 16: a group of GS lanes
// (GS = 8 or 16, GS >= n_t) owns one resource element, lane r owns row r of
// the n_t x n_t Hermitian Gram matrix A = H^H H in registers.  Two (GS = 16)
// or four (GS = 8) REs share a warp, so every lane is busy and the only
// shared memory per RE is H, y, the residual and three broadcast vectors.
//
// Same outputs and semantics as k_front in front.cu (which stays for
// 16 < n_t <= 32):
//   MMSE      linear.py:55-75      x = (A + s2 I)^-1 H^H y, projected; here by
//                                  Gauss-Jordan elimination (no pivoting; A + s2 I
//                                  is Hermitian positive definite, so its pivots
//                                  are the LDL^H pivots and "pivot <= 0" is
//                                  exactly cho_factor's failure condition)
//   Ising     transform.py:97-140  G = c^2 [[Re A, -Im A], [Im A, Re A]],
//                                  g = diag G, b = -c [Re; Im] H^H r,
//                                  offset = ||r||^2 + 2 tr G,
//   lambda_max transform.py:126    of G, i.e. of the Hermitian c^2 A whose rows
//                                  the lanes read back from the G they wrote:
//                                  Lanczos (n steps from a fixed irregular start
//                                  vector, stopping on an invariant subspace) to
//                                  a tridiagonal T, then Laguerre on the Sturm
//                                  polynomial of the (power-of-two scaled) T.
// One Gram per RE: its rows are written as G, then eliminated in place by
// the MMSE; lambda_max needs no copy of them (no global scratch).
#ifndef IL_FRONT_CPASYNC  // H, y staged by cp.async (0: through registers, 0.555 vs 0.540 ms)
#define IL_FRONT_CPASYNC 1
#endif
#include <float.h>

#include "il_group.cuh"
#include "il_internal.cuh"
#include "rng_numpy.cuh"

namespace il {

namespace {

constexpr int kRowsThreads = 128;
#ifndef IL_GRAM_UNROLL
#define IL_GRAM_UNROLL 1
#endif
constexpr int kGramUnroll = IL_GRAM_UNROLL;

// Per-group shared-memory slice (cplx units).
IL_HD size_t rows_group_cplx(int n_r, int n, int GS) {
    return (size_t)n_r * n + 2 * (size_t)n_r + 6 * (size_t)GS + 3 + 1;
}

// A row r = sum_k conj(H[k][r]) H[k][:] (zero rows/cols beyond n), z_r = (H^H y)_r.
// Im A is accumulated as two separate sums (sum hr.re hj.im) - (sum hr.im hj.re)
// so that A[j][r] == conj(A[r][j]) exactly (the diagonal's imaginary part is
// exactly zero) -- G is then exactly symmetric, as (G + G^T)/2 makes it in
// transform.py:123.
template <int GS>
__device__ __forceinline__ void gram_row(const cplx* H, const cplx* y, int n_r, int n, int r,
                                         cplx (&A)[GS], cplx* z) {
    double im2[GS];
#pragma unroll
    for (int j = 0; j < GS; ++j) A[j] = {0.0, 0.0}, im2[j] = 0.0;
    cplx zz = {0.0, 0.0};
    const bool own = r < n;
#pragma unroll kGramUnroll
    for (int k = 0; k < n_r; ++k) {
        const cplx* Hk = H + k * n;
        const cplx hr = own ? Hk[r] : cplx{0.0, 0.0};
#pragma unroll
        for (int j = 0; j < GS; ++j) {
            if (j < n) {
                const cplx hj = Hk[j];
                A[j].re = fma(hr.re, hj.re, fma(hr.im, hj.im, A[j].re));
                A[j].im = fma(hr.re, hj.im, A[j].im);
                im2[j] = fma(hr.im, hj.re, im2[j]);
            }
        }
        if (z) {
            const cplx yk = y[k];
            zz.re = fma(hr.re, yk.re, fma(hr.im, yk.im, zz.re));
            zz.im = fma(hr.re, yk.im, fma(-hr.im, yk.re, zz.im));
        }
    }
#pragma unroll
    for (int j = 0; j < GS; ++j) A[j].im -= im2[j];
    if (z) *z = zz;
}

// Exact power-of-two helpers (no frexp/ldexp software sequences).
IL_D int exp2_of(double m) {  // m in [2^(e-1), 2^e) -> e (frexp exponent), m > 0 normal
    return (int)((__double_as_longlong(m) >> 52) & 0x7ff) - 1022;
}
IL_D double pow2(int e) { return __longlong_as_double((long long)(1023 + e) << 52); }

// Largest eigenvalue of a symmetric tridiagonal matrix (diagonal dd[0..m),
// off-diagonal ee[0..m-1)), identical in every lane: Gershgorin bounds, an
// exact power-of-two scaling so that the Sturm recurrences cannot overflow
// (|P_k| <= 3^k) -- the iterates are those of the unscaled iteration -- and
// Laguerre's method from above on the characteristic polynomial, which
// converges monotonically (cubically) to the largest root.
template <int GS>
IL_D double tridiag_max(double (&dd)[GS], double (&ee)[GS], int m) {
    if (m == 1) return dd[0];
    double hi = -DBL_MAX, lo = DBL_MAX;
#pragma unroll
    for (int i = 0; i < GS; ++i) {
        if (i < m) {
            const double rr = (i > 0 ? ee[i - 1] : 0.0) + (i < m - 1 ? ee[i] : 0.0);
            hi = fmax(hi, dd[i] + rr);
            lo = fmin(lo, dd[i] - rr);
        }
    }
    double x = hi + 4.0 * DBL_EPSILON * fmax(fabs(hi), fabs(hi - lo)) + DBL_MIN;
    const int ex = exp2_of(fmax(fmax(fabs(hi), fabs(lo)), DBL_MIN));
    const double down = pow2(-ex);
#pragma unroll
    for (int i = 0; i < GS; ++i) {
        dd[i] *= down;
        ee[i] = (ee[i] * down) * (ee[i] * down);  // squared sub-diagonal
    }
    x *= down;
    const double nn = (double)m;
    for (int it = 0; it < 64; ++it) {
        double p0 = 1.0, p1 = 0.0, p2 = 0.0, q0 = 0.0, q1 = 0.0, q2 = 0.0;
#pragma unroll
        for (int k = 0; k < GS; ++k) {
            if (k < m) {
                const double dk = dd[k] - x;
                const double e2 = k > 0 ? ee[k - 1] : 0.0;
                const double r0 = dk * p0 - e2 * q0;
                const double r1 = dk * p1 - e2 * q1 - p0;
                const double r2 = dk * p2 - e2 * q2 - 2.0 * p1;
                q0 = p0; q1 = p1; q2 = p2;
                p0 = r0; p1 = r1; p2 = r2;
            }
        }
        if (p0 == 0.0) break;
        const double ip = 1.0 / p0;
        const double G = p1 * ip;
        const double Hh = G * G - p2 * ip;
        const double disc = fmax((nn - 1.0) * (nn * Hh - G * G), 0.0);
        const double den = G + sqrt(disc);
        if (!(den > 0.0)) break;
        const double step = nn / den;
        x -= step;
        if (!(step > 2.0 * DBL_EPSILON * fabs(x))) break;
    }
    return x * pow2(ex);
}

// Lanczos tridiagonalisation of the Hermitian matrix whose row r lives in
// lane r's B (kept): T_k = V^H B V over the Krylov space of a fixed start
// vector with irregular entries (a start vector orthogonal to the top
// eigenvector is as unlikely as for a random one); n steps, or fewer when the
// space becomes invariant (beta below 1e-14 of the row-sum norm; for B = c I
// or B = 0 after one step).  No reorthogonalisation is needed for the
// extreme Ritz value.  Emulated in numpy against LAPACK eigvalsh on 2x10^4
// 16x16 Wishart matrices: 2.6e-15 relative worst case (the Householder +
// Laguerre route this replaces took 2.5x the FP64 work).  vb: 2*GS-cplx
// broadcast buffer of the group; T goes to dsm (diagonal) and esm
// (sub-diagonal); returns its order m.
template <int GS>
__device__ int lanczos_rows(const Grp<GS>& g, const cplx (&Bm)[GS], int n, cplx* vb,
                            double* dsm, double* esm) {
    const int r = g.r;
    // start vector: (0.5 + frac((r+1) phi)) + i (0.5 + frac(3.1 (r+1) phi^2)), normalised
    cplx v = {0.0, 0.0};
    if (r < n) {
        const double phi = 0.6180339887498949;
        double ip;
        v = {0.5 + modf((r + 1) * phi, &ip), 0.5 + modf((r + 1) * phi * phi * 3.1, &ip)};
    }
    {
        const double inv = 1.0 / sqrt(g.sum(cabs2(v)));
        v = {v.re * inv, v.im * inv};
    }
    double nrm = 0.0;  // row-sum norm (scale of the breakdown test)
#pragma unroll
    for (int j = 0; j < GS; ++j) nrm += fabs(Bm[j].re) + fabs(Bm[j].im);
#pragma unroll
    for (int o = GS / 2; o > 0; o >>= 1) nrm = fmax(nrm, __shfl_xor_sync(g.mask, nrm, o, GS));
    cplx vp = {0.0, 0.0};
    double beta = 0.0;
    int m = n;
#pragma unroll 1
    for (int k = 0; k < n; ++k) {
        // v_k is broadcast through one of two halves of vb, alternating, so
        // that one group barrier per step separates writes from reads
        cplx* vk = vb + (k & 1) * GS;
        vk[r] = v;
        g.sync();
        // w = B v with the even and odd columns in separate accumulators
        // (half the dependent-FMA chain)
        cplx w0 = {0.0, 0.0}, w1 = {0.0, 0.0};
#pragma unroll
        for (int j = 0; j < GS; j += 2) {
            const cplx v0 = vk[j], v1 = vk[j + 1];
            w0.re = fma(Bm[j].re, v0.re, fma(-Bm[j].im, v0.im, w0.re));
            w0.im = fma(Bm[j].re, v0.im, fma(Bm[j].im, v0.re, w0.im));
            w1.re = fma(Bm[j + 1].re, v1.re, fma(-Bm[j + 1].im, v1.im, w1.re));
            w1.im = fma(Bm[j + 1].re, v1.im, fma(Bm[j + 1].im, v1.re, w1.im));
        }
        cplx w = {w0.re + w1.re, w0.im + w1.im};
        // alpha = v^H w and ||w||^2 in one reduction; then ||w'||^2 =
        // ||w||^2 - alpha^2 - beta^2 for w' = w - alpha v - beta v_prev
        // (exact for orthonormal v, v_prev), except where that difference
        // cancels (< 1% of ||w||^2: about 1% of the steps on Wishart
        // matrices, and every step of B = c I), which sums ||w'||^2 directly
        double a = v.re * w.re + v.im * w.im, ww = cabs2(w);
        g.sum2(a, ww);
        w = {w.re - a * v.re - beta * vp.re, w.im - a * v.im - beta * vp.im};
        if (r == 0) dsm[k] = a;
        double b2 = ww - a * a - beta * beta;
        if (!(b2 >= 0.01 * ww)) b2 = g.sum(cabs2(w));
        const double b = sqrt(b2);
        if (k == n - 1) break;
        if (!(b > 1e-14 * nrm)) {  // invariant subspace (or B = 0): T_{k+1} is exact
            m = k + 1;
            break;
        }
        if (r == 0) esm[k] = b;
        const double ib = 1.0 / b;
        vp = v;
        v = {w.re * ib, w.im * ib};
        beta = b;
    }
    g.sync();  // the last v_k has been read before vb is reused
    return m;
}

// Per-group slice: ... misc[2] holds the order m of the Lanczos tridiagonal
// T (d in dsm, e in esm) for the CTA's eigenvalue stage.
template <int GS, bool DO_MMSE, bool DO_ISING>
__device__ __forceinline__ void front_group(const Grp<GS>& g, int64_t prob, cplx* H,
                                            const double* __restrict__ Hg,
                                            const double* __restrict__ yg,
                                            const double* __restrict__ s2g, int n_r, int n,
                                            const Alphabet& al, uint8_t* __restrict__ x_idx,
                                            double* __restrict__ energy,
                                            int8_t* __restrict__ status, const IsingOut& o) {
    const int r = g.r;
    cplx* y = H + n_r * n;
    cplx* res = y + n_r;
    cplx* vb = res + n_r;
    cplx* wb = vb + 2 * GS;
    cplx* xs = wb + 2 * GS;    // decided symbols x_g (GS)
    cplx* misc = xs + GS;      // [0] = Gauss-Jordan rhs broadcast, [2].re = order of T
    double* dsm = reinterpret_cast<double*>(misc + 3);  // tridiagonal d[GS]
    double* esm = dsm + GS;                              // and e[GS]
    uint8_t* idx = x_idx + prob * 2 * n;
    {
        const cplx* Hp = reinterpret_cast<const cplx*>(Hg) + prob * (int64_t)n_r * n;
        const cplx* yp = reinterpret_cast<const cplx*>(yg) + prob * (int64_t)n_r;
#if IL_FRONT_CPASYNC
        // asynchronous 16-byte copies straight into shared memory: all of a
        // lane's loads in flight at once, no register staging
        for (int i = r; i < n_r * n; i += GS)
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"((uint32_t)__cvta_generic_to_shared(H + i)),
                         "l"(Hp + i)
                         : "memory");
        for (int i = r; i < n_r; i += GS)
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"((uint32_t)__cvta_generic_to_shared(y + i)),
                         "l"(yp + i)
                         : "memory");
        asm volatile("cp.async.wait_all;" ::: "memory");
#else
        for (int i = r; i < n_r * n; i += GS) H[i] = Hp[i];
        for (int i = r; i < n_r; i += GS) y[i] = yp[i];
#endif
    }
    g.sync();
    const double c = 0.5 * al.spacing;
    const double c2 = c * c;
    const int N = 2 * n;
    cplx A[GS];
    cplx zr;
    gram_row<GS>(H, y, n_r, n, r, A, &zr);
    double tr = 0.0;
    double gmax = 0.0, gsum = 0.0;  // max |G| and sum |G| over rows r, n + r (o.gstats)
    double* Gr = o.G + prob * (int64_t)N * N + (int64_t)r * N;  // G row r (valid for r < n)
    if (DO_ISING) {
        // G rows r and n + r (16-byte stores), g_diag, trace
        if (r < n) {
            double* Gs = Gr + (int64_t)n * N;
#pragma unroll
            for (int j = 0; j < GS; j += 2) {
                if (j + 1 < n && (n & 1) == 0) {  // 16-byte aligned only for even n
                    *reinterpret_cast<double2*>(Gr + j) = make_double2(c2 * A[j].re, c2 * A[j + 1].re);
                    *reinterpret_cast<double2*>(Gr + n + j) =
                        make_double2(c2 * -A[j].im, c2 * -A[j + 1].im);
                    *reinterpret_cast<double2*>(Gs + j) = make_double2(c2 * A[j].im, c2 * A[j + 1].im);
                    *reinterpret_cast<double2*>(Gs + n + j) =
                        make_double2(c2 * A[j].re, c2 * A[j + 1].re);
                } else {
#pragma unroll
                    for (int q = j; q < j + 2; ++q) {
                        if (q < n) {
                            Gr[q] = c2 * A[q].re;
                            Gr[n + q] = c2 * -A[q].im;
                            Gs[q] = c2 * A[q].im;
                            Gs[n + q] = c2 * A[q].re;
                        }
                    }
                }
            }
            if (o.gstats) {
                // the stored magnitudes: |c2 Re A|, |c2 Im A|, twice each
#pragma unroll
                for (int j = 0; j < GS; ++j) {
                    if (j < n) {
                        const double ar = fabs(c2 * A[j].re), ai = fabs(c2 * A[j].im);
                        gmax = fmax(gmax, fmax(ar, ai));
                        gsum += ar + ai;
                    }
                }
                gsum *= 2.0;
            }
            double arr = 0.0;
#pragma unroll
            for (int j = 0; j < GS; ++j)
                if (j == r) arr = A[j].re;
            const double gi = c2 * arr;
            if (o.g) {
                o.g[prob * N + r] = gi;
                o.g[prob * N + n + r] = gi;
            }
            tr = 2.0 * gi;
        }
        tr = g.sum(tr);
        // lambda_max(G) = c^2 lambda_max(A): Lanczos on the register rows of A
        // while they are intact (the MMSE below eliminates them in place); the
        // eigenvalue of T is taken by the CTA's last stage
        const int m = lanczos_rows<GS>(g, A, n, vb, dsm, esm);
        if (r == 0) misc[2].re = (double)m;
    }
    if (DO_MMSE) {
        const double s2 = s2g[prob];
#pragma unroll
        for (int j = 0; j < GS; ++j)
            if (j == r) A[j].re += s2;
        bool ok = true;
        cplx diag = {1.0, 0.0};
        // Gauss-Jordan, fully unrolled: at step k the pivot row's columns
        // k..GS-1 are broadcast through vb (and its rhs through misc), and
        // every other row eliminates column k, updating columns k+1.. only
        // (static register indices, trimmed loops: half the FP64 work of a
        // rolled loop over all columns)
        // (pivot rows alternate between the two halves of vb, their rhs
        // between misc[0] and misc[1]: one group barrier per step)
#pragma unroll
        for (int k = 0; k < GS; ++k) {
            if (k < n) {
                cplx* pk = vb + (k & 1) * GS;
                if (r == k) {
#pragma unroll
                    for (int j = k; j < GS; ++j) pk[j] = A[j];
                    misc[k & 1] = zr;
                }
                g.sync();
                const double piv = pk[k].re;
                ok = ok && (piv > 0.0);
                const double inv = 1.0 / piv;
                if (r == k) {
                    diag = A[k];
                } else {
                    const cplx f = {A[k].re * inv, A[k].im * inv};
#pragma unroll
                    for (int j = k + 1; j < GS; ++j) A[j] = csub(A[j], cmul(f, pk[j]));
                    zr = csub(zr, cmul(f, misc[k & 1]));
                }
            }
        }
        if (status && r == 0) status[prob] = ok ? 0 : -1;
        if (r < n) {
            const double inv = 1.0 / diag.re;
            const double xr = zr.re * inv, xi = zr.im * inv;
            const int kr = ok ? level_index(xr, al) : 0;
            const int ki = ok ? level_index(xi, al) : 0;
            idx[2 * r] = (uint8_t)kr;
            idx[2 * r + 1] = (uint8_t)ki;
            xs[r] = {al.levels[kr], al.levels[ki]};
        }
    } else if (r < n) {
        xs[r] = {al.levels[idx[2 * r]], al.levels[idx[2 * r + 1]]};
    }
    g.sync();

    // residual r = y - H x_g and ||r||^2 (linear.py:44-47).  The sum of the
    // |r_k|^2 is formed in exactly the order of a 32-lane warp_sum over
    // rows k = lane (+32, ...), the order k_select_decode uses for the
    // decoded vector, so that an unchanged decision reproduces E_guess
    // bit-for-bit and the strict test of detector.py:52 cannot flip.
    double acc = 0.0;
    for (int k = r; k < n_r; k += GS) res[k] = resid_row(H + k * n, xs, n, y[k]);
    g.sync();
    {
        double a[32 / GS];
#pragma unroll
        for (int q = 0; q < 32 / GS; ++q) {
            a[q] = 0.0;
            for (int k = r + q * GS; k < n_r; k += 32) a[q] = __dadd_rn(a[q], abs2_rn(res[k]));
        }
        // butterfly levels 16 (and 8 when GS = 8) of the 32-lane tree
        if (GS == 16) {
            acc = __dadd_rn(a[0], a[1]);
        } else {
            acc = __dadd_rn(__dadd_rn(a[0], a[2]), __dadd_rn(a[1], a[3]));
        }
    }
    const double r2 = g.sum(acc);
    if (energy && r == 0) energy[prob] = r2;
    if (DO_ISING) {
        g.sync();
        if (r < n) {
            double re = 0.0, im = 0.0;
            for (int k = 0; k < n_r; ++k) {
                const cplx h = H[k * n + r], v = res[k];
                re += h.re * v.re + h.im * v.im;
                im += h.re * v.im - h.im * v.re;
            }
            o.b[prob * N + r] = -c * re;
            o.b[prob * N + n + r] = -c * im;
            gsum += fabs(-c * re) + fabs(-c * im);
        }
        if (o.offset && r == 0) o.offset[prob] = r2 + 2.0 * tr;
        if (o.gstats) {
            // the anneal's operand scale and screen bound (k_anneal_fast)
#pragma unroll
            for (int q = GS / 2; q > 0; q >>= 1) gmax = fmax(gmax, __shfl_xor_sync(g.mask, gmax, q, GS));
            gsum = g.sum(gsum);
            if (r == 0) {
                o.gstats[2 * prob] = gmax;
                o.gstats[2 * prob + 1] = gsum;
            }
        }
    }
}

template <int GS, bool DO_MMSE, bool DO_ISING>
#ifndef IL_ROWS_MINB  // CTAs per SM for GS = 16 (3: 168 registers, no spills; 4 spills)
#define IL_ROWS_MINB 3
#endif
__global__ void __launch_bounds__(kRowsThreads, GS == 16 ? IL_ROWS_MINB : 4)
k_front_rows(const double* __restrict__ Hg, const double* __restrict__ yg,
             const double* __restrict__ s2g, int64_t P, int n_r, int n, Alphabet al,
             uint8_t* __restrict__ x_idx, double* __restrict__ energy,
             int8_t* __restrict__ status, IsingOut o) {
    extern __shared__ __align__(16) cplx smem_c[];
    constexpr int kGroups = kRowsThreads / GS;
    const size_t slice = rows_group_cplx(n_r, n, GS);
    {
        const Grp<GS> g;
        const int grp = threadIdx.x / GS;
        const int64_t prob = (int64_t)blockIdx.x * kGroups + grp;
        if (prob < P)  // whole groups together
            front_group<GS, DO_MMSE, DO_ISING>(g, prob, smem_c + grp * slice, Hg, yg, s2g, n_r, n, al,
                                               x_idx, energy, status, o);
    }
    if (!DO_ISING) return;
    // eigenvalue stage: lambda_max of each group's Lanczos tridiagonal, one
    // thread per resource element (the Laguerre iteration is sequential; run
    // once instead of redundantly in every lane of the group)
    __syncthreads();
    const int64_t prob = (int64_t)blockIdx.x * kGroups + threadIdx.x;
    if (threadIdx.x >= kGroups || prob >= P) return;
    const cplx* misc = smem_c + threadIdx.x * slice + (size_t)n_r * n + 2 * (size_t)n_r + 5 * GS;
    const double* dsm = reinterpret_cast<const double*>(misc + 3);
    const double* esm = dsm + GS;
    const int m = (int)misc[2].re;
    double dd[GS], ee[GS];
#pragma unroll
    for (int k = 0; k < GS; ++k) {
        dd[k] = k < m ? dsm[k] : 0.0;
        ee[k] = k + 1 < m ? esm[k] : 0.0;
    }
    const double c = 0.5 * al.spacing;
    const double lam = (c * c) * tridiag_max<GS>(dd, ee, m);
    const double S = (double)(4 * n + 1);
    const double es = 32.0 / sqrt(fmax(lam, 1e-30) * S);
    if (o.eps_scale) o.eps_scale[prob] = es;
    if (o.eps_out) o.eps_out[prob] = o.fixed_eps > 0.0 ? o.fixed_eps : es * o.eps_gain;
}

template <int GS, bool M, bool I>
int launch_rows_gs(const double* H, const double* y, const double* s2, int64_t P, int n_r, int n,
                   const Alphabet& al, uint8_t* x_idx, double* energy, int8_t* status,
                   const IsingOut& o, cudaStream_t st) {
    const int groups = kRowsThreads / GS;
    const size_t smem = sizeof(cplx) * rows_group_cplx(n_r, n, GS) * groups;
    auto fn = k_front_rows<GS, M, I>;
    IL_CHECK_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    const int64_t blocks = (P + groups - 1) / groups;
    IL_LAUNCH(kProfFront, st, fn<<<(unsigned)blocks, kRowsThreads, smem, st>>>(H, y, s2, P, n_r, n, al, x_idx, energy, status, o););
    IL_CHECK_CUDA(cudaGetLastError());
    return IL_OK;
}

}  // namespace

bool front_rows_supported(int n_r, int n_t) {
    if (n_t < 1 || n_t > 16 || n_r < 1) return false;
    const int GS = n_t <= 8 ? 8 : 16;
    return sizeof(cplx) * rows_group_cplx(n_r, n_t, GS) * (kRowsThreads / GS) <= 200 * 1024;
}

int launch_front_rows(bool do_mmse, bool do_ising, const double* H, const double* y,
                      const double* s2, int64_t P, int n_r, int n_t, const Alphabet& al,
                      uint8_t* x_idx, double* energy, int8_t* status, const IsingOut& o,
                      cudaStream_t st) {
    if (P == 0) return IL_OK;
    // H and y are staged by 16-byte cp.async copies
    IL_REQUIRE((((uintptr_t)H | (uintptr_t)y) & 15u) == 0,
               "H and y must be 16-byte aligned (complex128 device arrays)");
#define IL_ROWS(GS)                                                                                \
    do {                                                                                           \
        if (do_mmse && do_ising)                                                                   \
            return launch_rows_gs<GS, true, true>(H, y, s2, P, n_r, n_t, al, x_idx, energy, status, o, st); \
        if (do_mmse)                                                                               \
            return launch_rows_gs<GS, true, false>(H, y, s2, P, n_r, n_t, al, x_idx, energy, status, o, st); \
        return launch_rows_gs<GS, false, true>(H, y, s2, P, n_r, n_t, al, x_idx, energy, status, o, st); \
    } while (0)
    if (n_t <= 8) IL_ROWS(8);
    IL_ROWS(16);
#undef IL_ROWS
}

}  // namespace il
