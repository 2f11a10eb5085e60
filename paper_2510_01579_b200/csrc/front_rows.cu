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
//   lambda_max transform.py:126    Householder tridiagonalisation with rows in
//                                  registers, then Laguerre on the Sturm
//                                  polynomial of the (power-of-two scaled)
//                                  tridiagonal matrix.
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
#ifndef IL_ELIM_UNROLL  // unroll of the Householder / Gauss-Jordan step loops
#define IL_ELIM_UNROLL 1
#endif
constexpr int kElimUnroll = IL_ELIM_UNROLL;
#ifndef IL_PROBE_NO_LAMBDA
#define IL_PROBE_NO_LAMBDA 0
#endif
#ifndef IL_PROBE_FRONT_RNG
#define IL_PROBE_FRONT_RNG 0
#endif
#ifndef IL_FRONT_TMA  // H, y staged by TMA bulk copies
#define IL_FRONT_TMA 0  // measured slower: 0.80 -> 1.22 ms per 16x16 slot
#endif
#ifndef IL_FRONT_SAVE_A  // phase 1 reloads the Gram rows instead of recomputing them
#define IL_FRONT_SAVE_A 1
#endif

// Per-group shared-memory slice (cplx units).
IL_HD size_t rows_group_cplx(int n_r, int n, int GS) {
    return (size_t)n_r * n + 2 * (size_t)n_r + 6 * (size_t)GS + 2 + 1;
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

// Drop column 0 of the lane's row: A[j] <- A[j + 1].  Keeping the active
// column at index 0 lets the elimination loops stay rolled (small code, no
// instruction-cache thrash) while every register index is static.
template <int GS>
IL_D void shift_row(cplx (&A)[GS]) {
#pragma unroll
    for (int j = 0; j + 1 < GS; ++j) A[j] = A[j + 1];
    A[GS - 1] = {0.0, 0.0};
}

// Largest eigenvalue of the Hermitian matrix whose row r lives in lane r's A
// (destroyed).  vb, wb: 2*GS-cplx broadcast buffers of the group whose upper
// halves are zero; dsm, esm: GS-double tridiagonal scratch.
template <int GS>
__device__ double lambda_max_rows(const Grp<GS>& g, cplx (&A)[GS], int n, cplx* vb, cplx* wb,
                                  double* dsm, double* esm) {
    const int r = g.r;
    // Householder tridiagonalisation; at step k, A[j] holds column k + j.
#pragma unroll kElimUnroll
    for (int k = 0; k + 2 < n; ++k) {
        const cplx xi = (r > k && r < n) ? A[0] : cplx{0.0, 0.0};
        const double sig2 = g.sum(cabs2(xi));
        if (r == k) dsm[k] = A[0].re;
        const cplx x0 = g.bcast(xi, k + 1);
        double tau = 0.0, sig = 0.0;
        cplx ph = {1.0, 0.0};
        if (sig2 > 0.0) {
            sig = sqrt(sig2);
            const double ax0 = sqrt(cabs2(x0));
            if (ax0 > 0.0) {
                const double ia = 1.0 / ax0;
                ph = {x0.re * ia, x0.im * ia};
            }
            tau = 1.0 / (sig * (sig + ax0));
        }
        if (r == 0) esm[k] = sig;
        const cplx vr = (r == k + 1) ? cplx{xi.re + ph.re * sig, xi.im + ph.im * sig} : xi;
        vb[r] = vr;
        g.sync();
        const cplx* vk = vb + k;
        const cplx* wk = wb + k;
        cplx p = {0.0, 0.0};
#pragma unroll
        for (int j = 1; j < GS; ++j) p = cadd(p, cmul(A[j], vk[j]));
        p = {tau * p.re, tau * p.im};
        const double vhp = g.sum(vr.re * p.re + vr.im * p.im);
        const double K = 0.5 * tau * vhp;
        const cplx wr = {p.re - K * vr.re, p.im - K * vr.im};
        wb[r] = wr;
        g.sync();
#pragma unroll
        for (int j = 1; j < GS; ++j) {
            const cplx vj = vk[j], wj = wk[j];
            // B[r][j] -= v_r conj(w_j) + w_r conj(v_j)
            A[j] = csub(A[j], cadd(cmulc(wj, vr), cmulc(vj, wr)));
        }
        shift_row<GS>(A);
        g.sync();  // vb/wb are rewritten by the next step
    }
    // trailing 2x2 (A[j] holds column max(n-2, 0) + j): rows n-2 and n-1
    if (n >= 2) {
        if (r == n - 2) dsm[n - 2] = A[0].re;
        if (r == n - 1) {
            dsm[n - 1] = A[1].re;
            esm[n - 2] = sqrt(cabs2(A[0]));
        }
    } else if (r == 0) {
        dsm[0] = A[0].re;
    }
    g.sync();
    if (n == 1) return dsm[0];
    double dd[GS], ee[GS];
#pragma unroll
    for (int k = 0; k < GS; ++k) {
        dd[k] = k < n ? dsm[k] : 0.0;
        ee[k] = k + 1 < n ? esm[k] : 0.0;
    }

    // Gershgorin bounds, then an exact power-of-two scaling so that the
    // Sturm recurrences cannot overflow (|P_k| <= 3^k) -- the iterates are
    // those of the unscaled iteration.
    double hi = -DBL_MAX, lo = DBL_MAX;
#pragma unroll
    for (int i = 0; i < GS; ++i) {
        if (i < n) {
            const double rr = (i > 0 ? ee[i - 1] : 0.0) + (i < n - 1 ? ee[i] : 0.0);
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
    const double nn = (double)n;
    for (int it = 0; it < 64; ++it) {
        double p0 = 1.0, p1 = 0.0, p2 = 0.0, q0 = 0.0, q1 = 0.0, q2 = 0.0;
#pragma unroll
        for (int k = 0; k < GS; ++k) {
            if (k < n) {
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

template <int GS, bool DO_MMSE, bool DO_ISING>
#ifndef IL_ROWS_MINB
#define IL_ROWS_MINB 4
#endif
__global__ void __launch_bounds__(kRowsThreads, IL_ROWS_MINB)
k_front_rows(const double* __restrict__ Hg, const double* __restrict__ yg,
             const double* __restrict__ s2g, int64_t P, int n_r, int n, Alphabet al,
             uint8_t* __restrict__ x_idx, double* __restrict__ energy,
             int8_t* __restrict__ status, IsingOut o, cplx* __restrict__ ascratch) {
    extern __shared__ __align__(16) cplx smem_c[];
    const Grp<GS> g;
    const int r = g.r;
    const int grp = threadIdx.x / GS;
    const int64_t prob = (int64_t)blockIdx.x * (kRowsThreads / GS) + grp;
    if (prob >= P) return;  // whole groups exit together
    cplx* H = smem_c + grp * rows_group_cplx(n_r, n, GS);
    cplx* y = H + n_r * n;
    cplx* res = y + n_r;
    cplx* vb = res + n_r;
    cplx* wb = vb + 2 * GS;
    cplx* xs = wb + 2 * GS;    // decided symbols x_g (GS)
    cplx* misc = xs + GS;      // [0] = Gauss-Jordan rhs broadcast
    double* dsm = reinterpret_cast<double*>(misc + 2);  // tridiagonal d[GS]
    double* esm = dsm + GS;                              // and e[GS]
    uint8_t* idx = x_idx + prob * 2 * n;
    {
        const cplx* Hp = reinterpret_cast<const cplx*>(Hg) + prob * (int64_t)n_r * n;
        const cplx* yp = reinterpret_cast<const cplx*>(yg) + prob * (int64_t)n_r;
#if IL_FRONT_TMA
        // H and y by 1-D TMA bulk copies (one lane of the group issues, every
        // lane waits on the group's mbarrier): no per-lane load loop whose
        // iterations each wait out a DRAM round trip
        __shared__ __align__(8) uint64_t bars[kRowsThreads / GS];
        uint64_t* bar = &bars[grp];
        if (r == 0) {
            mbar_init(bar, 1);
            asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
            const uint32_t hb = (uint32_t)(sizeof(cplx) * n_r * n), yb = (uint32_t)(sizeof(cplx) * n_r);
            mbar_expect_tx(bar, hb + yb);
            tma_bulk_g2s(H, Hp, hb, bar);
            tma_bulk_g2s(y, yp, yb, bar);
        }
        vb[GS + r] = wb[GS + r] = cplx{0.0, 0.0};  // zero tails read by shifted columns
        g.sync();
        mbar_wait(bar, 0);
#else
        for (int i = r; i < n_r * n; i += GS) H[i] = Hp[i];
        for (int i = r; i < n_r; i += GS) y[i] = yp[i];
        vb[GS + r] = wb[GS + r] = cplx{0.0, 0.0};  // zero tails read by shifted columns
#endif
    }
    g.sync();
    const double c = 0.5 * al.spacing;
    const double c2 = c * c;
    const int N = 2 * n;
    cplx A[GS];
    double tr = 0.0;
    // phase 0 (Ising): Gram -> G, g, tr G, lambda_max;  phase 1 (MMSE): Gram -> solve.
    // One rolled loop keeps a single copy of the Gram code.
    // with both phases, the Gram rows of phase 0 (destroyed by lambda_max)
    // are parked in global scratch, [prob][j][r] so that a store or load of
    // one column is 16 consecutive lanes, and phase 1 reloads them
    cplx* asv = (DO_MMSE && DO_ISING && ascratch) ? ascratch + prob * (int64_t)GS * GS + r : nullptr;
    cplx zr;
#pragma unroll 1
    for (int phase = DO_ISING ? 0 : 1; phase < (DO_MMSE ? 2 : 1); ++phase) {
        if (phase == 1 && asv) {
#pragma unroll
            for (int j = 0; j < GS; ++j) A[j] = asv[j * GS];
        } else {
            gram_row<GS>(H, y, n_r, n, r, A, &zr);
            if (phase == 0 && asv) {
#pragma unroll
                for (int j = 0; j < GS; ++j) asv[j * GS] = A[j];
            }
        }
        if (phase == 0) {
            // G rows r and n + r (16-byte stores), g_diag, trace
            if (r < n) {
                double* Gr = o.G + prob * (int64_t)N * N + (int64_t)r * N;
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
#if IL_PROBE_NO_LAMBDA  // timing probe only: skips lambda_max (wrong eps)
            const double lam_a = 1.0;
#else
            const double lam_a = lambda_max_rows<GS>(g, A, n, vb, wb, dsm, esm);
#endif
            if (r == 0) {
                const double lam = c2 * lam_a;
                const double S = (double)(2 * N + 1);
                const double es = 32.0 / sqrt(fmax(lam, 1e-30) * S);
                if (o.eps_scale) o.eps_scale[prob] = es;
                if (o.eps_out) o.eps_out[prob] = o.fixed_eps > 0.0 ? o.fixed_eps : es * o.eps_gain;
            }
        } else {
            const double s2 = s2g[prob];
#pragma unroll
            for (int j = 0; j < GS; ++j)
                if (j == r) A[j].re += s2;
            bool ok = true;
            cplx diag = {1.0, 0.0};
            // Gauss-Jordan: pivot row k broadcast through vb (row) and misc (rhs);
            // at step k, A[j] holds column k + j
#pragma unroll kElimUnroll
            for (int k = 0; k < n; ++k) {
                if (r == k) {
#pragma unroll
                    for (int j = 0; j < GS; ++j) vb[j] = A[j];
                    misc[0] = zr;
                }
                g.sync();
                const double piv = vb[0].re;
                ok = ok && (piv > 0.0);
                const double inv = 1.0 / piv;
                if (r == k) {
                    diag = A[0];
                } else {
                    const cplx f = {A[0].re * inv, A[0].im * inv};
#pragma unroll
                    for (int j = 1; j < GS; ++j) A[j] = csub(A[j], cmul(f, vb[j]));
                    zr = csub(zr, cmul(f, misc[0]));
                }
                shift_row<GS>(A);
                g.sync();
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
        }
    }
    if (!DO_MMSE && r < n) xs[r] = {al.levels[idx[2 * r]], al.levels[idx[2 * r + 1]]};
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
        }
        if (o.offset && r == 0) o.offset[prob] = r2 + 2.0 * tr;
#if IL_PROBE_FRONT_RNG
        // timing probe only: the x0 replay of the anneal kernel (32 anneals x
        // 2n+1... here 65 draws each, 2 per lane-anneal chain) done here
        // instead; written over G (wrong results)
        {
            constexpr int kS = 65;
            for (int a = r; a < 32; a += GS) {
                Pcg64 rng;
                rng.seed_from(derive_seed2((uint64_t)prob * 977u, (uint64_t)a));
                float* dst = reinterpret_cast<float*>(o.G + prob * (int64_t)N * N) + a * kS;
                for (int i = 0; i < kS; ++i) dst[i] = (float)rng.uniform(-0.1, 0.2);
            }
        }
#endif
    }
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
    cplx* scratch = nullptr;
    if (M && I && IL_FRONT_SAVE_A)
        if (const int rc = pool_alloc((void**)&scratch, sizeof(cplx) * GS * GS * (size_t)P, st)) return rc;
    IL_LAUNCH(kProfFront, st, fn<<<(unsigned)blocks, kRowsThreads, smem, st>>>(H, y, s2, P, n_r, n, al, x_idx, energy, status, o, scratch););
    const cudaError_t e = cudaGetLastError();
    if (scratch) cudaFreeAsync(scratch, st);
    IL_CHECK_CUDA(e);
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
