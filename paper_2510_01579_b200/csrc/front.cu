// FP64 per-problem reduction kernels: MMSE front-end, Ising reduction with
// lambda_max, ZF/VPP front-end, and the selection/decode epilogue.
//
// One warp owns one problem (a resource element); its matrices live in a
// warp-private slice of shared memory, lanes own rows.  Everything here is
// FP64 because the hard decisions must match the reference: an FP32 MMSE
// flips 1-3 decisions per 10^4 REs at 16x16.
//
// Reference map:
//   mmse front      linear.py:55-75        (A = H^H H + s2 I, Cholesky solve, project)
//   build_ising     transform.py:97-140    (G, g_diag, b, offset, eps_scale)
//   lambda_max      transform.py:126       (eigvalsh(G)[-1] = c^2 lambda_max(H^H H))
//   zf / vpp front  precoder.py:54-60, 93-125
//   select/decode   solver.py:256-279, detector.py:44-54, transform.py:155-169
//   vpp post        precoder.py:126-146
#include <float.h>

#include <algorithm>

#include "il_internal.cuh"
#include "rng_numpy.cuh"

namespace il {

namespace {

constexpr unsigned kFull = 0xffffffffu;

// ---------------------------------------------------------------------------
// warp-cooperative FP64 linear algebra on shared-memory matrices (row-major)
// ---------------------------------------------------------------------------

// A[n_t x n_t] = H^H H (exactly Hermitian: upper half computed, mirrored),
// z[n_t] = H^H y.  H is [n_r x n_t].
__device__ void gram_hermitian(const cplx* H, const cplx* y, int n_r, int n_t, cplx* A, cplx* z,
                               int lane) {
    for (int idx = lane; idx < n_t * n_t; idx += 32) {
        const int i = idx / n_t, j = idx % n_t;
        if (i > j) continue;
        double re = 0.0, im = 0.0;
        for (int k = 0; k < n_r; ++k) {
            const cplx hi = H[k * n_t + i], hj = H[k * n_t + j];
            re += hi.re * hj.re + hi.im * hj.im;
            im += hi.re * hj.im - hi.im * hj.re;
        }
        if (i == j) im = 0.0;
        A[i * n_t + j] = {re, im};
        A[j * n_t + i] = {re, -im};
    }
    if (y) {
        for (int i = lane; i < n_t; i += 32) {
            double re = 0.0, im = 0.0;
            for (int k = 0; k < n_r; ++k) {
                const cplx h = H[k * n_t + i], v = y[k];
                re += h.re * v.re + h.im * v.im;
                im += h.re * v.im - h.im * v.re;
            }
            z[i] = {re, im};
        }
    }
    __syncwarp();
}

// In-place lower Cholesky M = L L^H (M Hermitian positive definite, n <= 32,
// lane i owns row i); inv_diag[k] = 1 / L[k][k] (scaling by the reciprocal,
// as LAPACK's zpotrf does).  Returns false on a non-positive pivot (the
// reference raises LinAlgError from cho_factor in that case).
template <unsigned GMASK_ALL = 0>
__device__ bool cholesky_lower_g(cplx* M, int n, double* inv_diag, int lane, unsigned mask) {
    // lane: index within the group that owns M; mask: the group's warp lanes
    for (int k = 0; k < n; ++k) {
        const double piv = M[k * n + k].re;
        if (!(piv > 0.0)) return false;
        const double lkk = sqrt(piv);
        const double inv = 1.0 / lkk;
        __syncwarp(mask);
        cplx lik = {0.0, 0.0};
        if (lane > k && lane < n) {
            const cplx v = M[lane * n + k];
            lik = {v.re * inv, v.im * inv};
            M[lane * n + k] = lik;
        }
        if (lane == k) {
            M[k * n + k] = {lkk, 0.0};
            inv_diag[k] = inv;
        }
        __syncwarp(mask);
        if (lane > k && lane < n) {
            for (int j = k + 1; j <= lane; ++j) {
                const cplx ljk = M[j * n + k];
                M[lane * n + j].re -= lik.re * ljk.re + lik.im * ljk.im;
                M[lane * n + j].im -= lik.im * ljk.re - lik.re * ljk.im;
            }
        }
        __syncwarp(mask);
    }
    return true;
}

__device__ bool cholesky_lower(cplx* M, int n, double* inv_diag, int lane) {
    for (int k = 0; k < n; ++k) {
        const double piv = M[k * n + k].re;
        if (!(piv > 0.0)) return false;
        const double lkk = sqrt(piv);
        const double inv = 1.0 / lkk;
        __syncwarp();
        cplx lik = {0.0, 0.0};
        if (lane > k && lane < n) {
            const cplx v = M[lane * n + k];
            lik = {v.re * inv, v.im * inv};
            M[lane * n + k] = lik;
        }
        if (lane == k) {
            M[k * n + k] = {lkk, 0.0};
            inv_diag[k] = inv;
        }
        __syncwarp();
        if (lane > k && lane < n) {
            for (int j = k + 1; j <= lane; ++j) {
                const cplx ljk = M[j * n + k];
                // M[i][j] -= L[i][k] * conj(L[j][k])
                M[lane * n + j].re -= lik.re * ljk.re + lik.im * ljk.im;
                M[lane * n + j].im -= lik.im * ljk.re - lik.re * ljk.im;
            }
        }
        __syncwarp();
    }
    return true;
}

// Solve (L L^H) x = rhs in place (rhs -> x); L lower from cholesky_lower.
__device__ void cholesky_solve(const cplx* L, const double* inv_diag, int n, cplx* x, int lane) {
    cplx xl = lane < n ? x[lane] : cplx{0.0, 0.0};
    for (int k = 0; k < n; ++k) {  // L w = rhs (column sweep, rhs kept in registers)
        const double inv = inv_diag[k];
        const cplx xk = {__shfl_sync(kFull, xl.re, k) * inv, __shfl_sync(kFull, xl.im, k) * inv};
        if (lane == k) xl = xk;
        if (lane > k && lane < n) xl = csub(xl, cmul(L[lane * n + k], xk));
    }
    for (int k = n - 1; k >= 0; --k) {  // L^H x = w
        const double inv = inv_diag[k];
        const cplx xk = {__shfl_sync(kFull, xl.re, k) * inv, __shfl_sync(kFull, xl.im, k) * inv};
        if (lane == k) xl = xk;
        if (lane < k) xl = csub(xl, cmulc(L[k * n + lane], xk));
    }
    if (lane < n) x[lane] = xl;
    __syncwarp();
}

// Largest eigenvalue of the real symmetric tridiagonal T (diagonal d[0..n),
// off-diagonal e[0..n-1)), identical in every lane.
__device__ double tridiag_max_smem(const double* d, const double* e, int n) {
    if (n == 1) return d[0];
    // Largest root of det(T - x I) by Laguerre iteration from the Gershgorin
    // upper bound: for a polynomial with only real roots it converges
    // monotonically from above to the largest root, cubically (and exactly
    // in one step for a single multiple root).  Three-term recurrences give
    // p, p', p'' without divisions; every lane iterates redundantly.
    double hi = -DBL_MAX, lo = DBL_MAX;
    for (int i = 0; i < n; ++i) {
        const double r = (i > 0 ? e[i - 1] : 0.0) + (i < n - 1 ? e[i] : 0.0);
        hi = fmax(hi, d[i] + r);
        lo = fmin(lo, d[i] - r);
    }
    double x = hi + 4.0 * DBL_EPSILON * fmax(fabs(hi), fabs(hi - lo)) + DBL_MIN;
    const double nn = (double)n;
    for (int it = 0; it < 64; ++it) {
        double p0 = 1.0, p1 = 0.0, p2 = 0.0;      // P_{k-1}, P'_{k-1}, P''_{k-1}
        double q0 = 0.0, q1 = 0.0, q2 = 0.0;      // P_{k-2}, ...
        for (int k = 0; k < n; ++k) {
            const double dk = d[k] - x;
            const double e2 = k > 0 ? e[k - 1] * e[k - 1] : 0.0;
            const double r0 = dk * p0 - e2 * q0;
            const double r1 = dk * p1 - e2 * q1 - p0;
            const double r2 = dk * p2 - e2 * q2 - 2.0 * p1;
            q0 = p0; q1 = p1; q2 = p2;
            p0 = r0; p1 = r1; p2 = r2;
            const double mag = fabs(p0);
            if (mag > 1e150 || (mag < 1e-150 && mag > 0.0)) {
                const double sc = mag > 1e150 ? 1e-150 : 1e150;
                p0 *= sc; p1 *= sc; p2 *= sc; q0 *= sc; q1 *= sc; q2 *= sc;
            }
        }
        if (p0 == 0.0) break;  // landed on the root
        const double G = p1 / p0;
        const double Hh = G * G - p2 / p0;
        const double disc = fmax((nn - 1.0) * (nn * Hh - G * G), 0.0);
        const double den = G + sqrt(disc);
        if (!(den > 0.0)) break;
        const double step = nn / den;
        x -= step;
        if (!(step > 2.0 * DBL_EPSILON * fabs(x))) break;
    }
    return x;
}

// Largest eigenvalue of the Hermitian W[n x n] (read only, n <= 32): n Lanczos
// steps over the warp (lane r owns component r; W is read by columns, W[j][r]
// = conj(W[r][j]), so that the lanes' loads are consecutive), no
// reorthogonalisation (the extreme Ritz value converges regardless), then
// the Laguerre iteration on the tridiagonal.  The same start vector and
// breakdown rule as the row front end's lanczos_rows (front_rows.cu).
// Replaces a Householder reduction (2.5x the FP64 work, n - 2 rank-2 updates
// of the shared-memory matrix).  scratch: n cplx + 2n double.
__device__ double lambda_max_hermitian(const cplx* W, int n, cplx* scratch, int lane) {
    cplx* vb = scratch;
    double* d = reinterpret_cast<double*>(scratch + n);
    double* e = d + n;
    const bool own = lane < n;
    cplx v = {0.0, 0.0};
    double nrm = 0.0;  // row-sum norm (scale of the breakdown test)
    if (own) {
        const double phi = 0.6180339887498949;
        double ip;
        v = {0.5 + modf((lane + 1) * phi, &ip), 0.5 + modf((lane + 1) * phi * phi * 3.1, &ip)};
        for (int j = 0; j < n; ++j) nrm += fabs(W[j * n + lane].re) + fabs(W[j * n + lane].im);
    }
    {
        const double inv = 1.0 / sqrt(warp_sum(cabs2(v)));
        v = {v.re * inv, v.im * inv};
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) nrm = fmax(nrm, __shfl_xor_sync(0xffffffffu, nrm, o));
    cplx vp = {0.0, 0.0};
    double beta = 0.0;
    int m = n;
    for (int k = 0; k < n; ++k) {
        __syncwarp();  // the previous step's reads of vb are done
        if (own) vb[lane] = v;
        __syncwarp();
        cplx w0 = {0.0, 0.0}, w1 = {0.0, 0.0};
        if (own) {
            int j = 0;
            for (; j + 1 < n; j += 2) {
                const cplx a0 = W[j * n + lane], a1 = W[(j + 1) * n + lane];
                const cplx v0 = vb[j], v1 = vb[j + 1];
                w0 = cadd(w0, cmulc(a0, v0));  // conj(W[j][r]) v_j = W[r][j] v_j
                w1 = cadd(w1, cmulc(a1, v1));
            }
            if (j < n) w0 = cadd(w0, cmulc(W[j * n + lane], vb[j]));
        }
        cplx w = cadd(w0, w1);
        const double a = warp_sum(v.re * w.re + v.im * w.im);
        const double ww = warp_sum(cabs2(w));
        w = {w.re - a * v.re - beta * vp.re, w.im - a * v.im - beta * vp.im};
        if (lane == 0) d[k] = a;
        double b2 = ww - a * a - beta * beta;
        if (!(b2 >= 0.01 * ww)) b2 = warp_sum(cabs2(w));
        const double bk = sqrt(b2);
        if (k == n - 1) break;
        if (!(bk > 1e-14 * nrm)) {  // invariant subspace: T_{k+1} is exact
            m = k + 1;
            break;
        }
        if (lane == 0) e[k] = bk;
        const double ib = 1.0 / bk;
        vp = v;
        v = {w.re * ib, w.im * ib};
        beta = bk;
    }
    __syncwarp();
    return tridiag_max_smem(d, e, m);
}

// Per-warp shared-memory carve-up for the detection front-end.
struct FrontSmem {
    cplx *H, *y, *A, *z, *r, *scr;
    IL_HD static size_t bytes(int n_r, int n_t) {
        const size_t c = (size_t)n_r * n_t + n_r + (size_t)n_t * n_t + n_t + n_r + 5 * n_t + 4;
        return c * sizeof(cplx);
    }
    __device__ void carve(char* base, int n_r, int n_t) {
        H = reinterpret_cast<cplx*>(base);
        y = H + n_r * n_t;
        A = y + n_r;
        z = A + n_t * n_t;
        r = z + n_t;
        scr = r + n_r;
    }
};

__device__ void load_problem(const double* Hg, const double* yg, int64_t prob, int n_r, int n_t,
                             cplx* H, cplx* y, int lane) {
    const cplx* Hp = reinterpret_cast<const cplx*>(Hg) + prob * (int64_t)n_r * n_t;
    for (int i = lane; i < n_r * n_t; i += 32) H[i] = Hp[i];
    const cplx* yp = reinterpret_cast<const cplx*>(yg) + prob * (int64_t)n_r;
    for (int i = lane; i < n_r; i += 32) y[i] = yp[i];
    __syncwarp();
}

// r = y - H x_g (x_g from level indices), returns ||r||^2 on every lane.
__device__ double residual_from_idx(const cplx* H, const cplx* y, const uint8_t* idx, int n_r,
                                    int n_t, const Alphabet& al, cplx* r, cplx* xs, int lane) {
    for (int j = lane; j < n_t; j += 32) xs[j] = {al.levels[idx[2 * j]], al.levels[idx[2 * j + 1]]};
    __syncwarp();
    double acc = 0.0;
    for (int k = lane; k < n_r; k += 32) {
        const cplx rk = resid_row(H + k * n_t, xs, n_t, y[k]);
        r[k] = rk;
        acc = __dadd_rn(acc, abs2_rn(rk));
    }
    __syncwarp();
    return warp_sum(acc);
}

// G and g_diag from the Gram matrix A (transform.py:108-140); returns tr(G)
// on every lane.
__device__ double emit_g(const cplx* A, int n_t, const Alphabet& al, int64_t prob,
                         const IsingOut& o, int lane) {
    const int N = 2 * n_t;
    const double c = 0.5 * al.spacing;
    const double c2 = c * c;
    double* G = o.G + prob * (int64_t)N * N;
    for (int idx = lane; idx < N * N; idx += 32) {
        const int i = idx / N, j = idx % N;
        const cplx aij = A[(i % n_t) * n_t + (j % n_t)];
        double v;
        if ((i < n_t) == (j < n_t)) v = aij.re;
        else v = (i < n_t) ? -aij.im : aij.im;
        G[idx] = c2 * v;
    }
    double tr = 0.0;
    for (int i = lane; i < n_t; i += 32) {
        const double gi = c2 * A[i * n_t + i].re;
        if (o.g) {
            o.g[prob * N + i] = gi;
            o.g[prob * N + n_t + i] = gi;
        }
        tr += 2.0 * gi;
    }
    return warp_sum(tr);
}

// b, offset and eps_scale around the guess whose residual is r (r2 =
// ||r||^2); lambda_max is taken of c^2 A as stored in G (its blocks [[Re,
// -Im], [Im, Re]] read back into the shared-memory slot W, so that A itself
// may have been factorised in place by then).
__device__ void emit_rest(const cplx* H, const cplx* r, double r2, double trg, cplx* W, cplx* scr,
                          int n_r, int n_t, const Alphabet& al, int64_t prob, const IsingOut& o,
                          int lane) {
    const int N = 2 * n_t;
    const double c = 0.5 * al.spacing;
    for (int i = lane; i < n_t; i += 32) {
        // H^H r
        double re = 0.0, im = 0.0;
        for (int k = 0; k < n_r; ++k) {
            const cplx h = H[k * n_t + i], v = r[k];
            re += h.re * v.re + h.im * v.im;
            im += h.re * v.im - h.im * v.re;
        }
        o.b[prob * N + i] = -c * re;
        o.b[prob * N + n_t + i] = -c * im;
    }
    const double* G = o.G + prob * (int64_t)N * N;
    __syncwarp();  // this warp's G stores are visible to its loads
    for (int idx = lane; idx < n_t * n_t; idx += 32) {
        const int i = idx / n_t, j = idx % n_t;
        W[idx] = {G[i * N + j], G[(n_t + i) * N + j]};
    }
    __syncwarp();
    const double lam = lambda_max_hermitian(W, n_t, scr, lane);
    if (lane == 0) {
        if (o.offset) o.offset[prob] = r2 + 2.0 * trg;  // ||r||^2 + 2 tr G
        const double S = (double)(2 * N + 1);
        const double es = 32.0 / sqrt(fmax(lam, 1e-30) * S);
        if (o.eps_scale) o.eps_scale[prob] = es;
        if (o.eps_out) o.eps_out[prob] = o.fixed_eps > 0.0 ? o.fixed_eps : es * o.eps_gain;
    }
    __syncwarp();
}

// Detection front-end.  DO_MMSE: guess = projected MMSE solution (written to
// x_idx, energy); else guess read from x_idx.  DO_ISING: emit the Ising problem.
template <bool DO_MMSE, bool DO_ISING>
__global__ void k_front(const double* __restrict__ Hg, const double* __restrict__ yg,
                        const double* __restrict__ s2g, int64_t P, int n_r, int n_t, Alphabet al,
                        uint8_t* __restrict__ x_idx, double* __restrict__ energy,
                        int8_t* __restrict__ status, IsingOut o) {
    extern __shared__ __align__(16) char smem_raw[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t prob = (int64_t)blockIdx.x * (blockDim.x >> 5) + warp;
    if (prob >= P) return;
    FrontSmem sm;
    sm.carve(smem_raw + warp * FrontSmem::bytes(n_r, n_t), n_r, n_t);
    load_problem(Hg, yg, prob, n_r, n_t, sm.H, sm.y, lane);
    gram_hermitian(sm.H, sm.y, n_r, n_t, sm.A, sm.z, lane);
    uint8_t* idx = x_idx + prob * 2 * n_t;
    // G first, so that the MMSE may factorise A in place (no second n_t^2 slot:
    // more warps per SM for these large shapes)
    const double trg = DO_ISING ? emit_g(sm.A, n_t, al, prob, o, lane) : 0.0;
    __syncwarp();  // every lane's reads of A precede the in-place factorisation
    if (DO_MMSE) {
        const double s2 = s2g[prob];
        for (int i = lane; i < n_t; i += 32) sm.A[i * n_t + i].re += s2;
        __syncwarp();
        double* invd = reinterpret_cast<double*>(sm.scr);
        const bool ok = cholesky_lower(sm.A, n_t, invd, lane);
        if (status && lane == 0) status[prob] = ok ? 0 : -1;
        if (ok) {
            cholesky_solve(sm.A, invd, n_t, sm.z, lane);
            for (int j = lane; j < n_t; j += 32) {
                idx[2 * j] = (uint8_t)level_index(sm.z[j].re, al);
                idx[2 * j + 1] = (uint8_t)level_index(sm.z[j].im, al);
            }
        } else {
            for (int j = lane; j < 2 * n_t; j += 32) idx[j] = 0;
        }
        __syncwarp();
    }
    const double r2 = residual_from_idx(sm.H, sm.y, idx, n_r, n_t, al, sm.r, sm.scr, lane);
    if (energy && lane == 0) energy[prob] = r2;
    if (DO_ISING) emit_rest(sm.H, sm.r, r2, trg, sm.A, sm.scr, n_r, n_t, al, prob, o, lane);
}

int front_blocks(int64_t P, size_t per_warp, int* wpb, size_t* smem) {
    // warps per CTA (4, 2 or 1) that fit the most warps per SM into its
    // 227 KB of shared memory (1 KB reserved per CTA): for n_t = 28, 1-warp
    // CTAs hold 7 warps per SM where 4-warp CTAs held 4
    const size_t sm_bytes = 227 * 1024;
    int w = 1, best = 0;
    for (int c : {4, 2, 1}) {
        if (c * per_warp > 200 * 1024) continue;
        const int ctas = (int)(sm_bytes / (c * per_warp + 1024));
        const int warps = std::min(ctas * c, 48);
        if (warps > best) {
            best = warps;
            w = c;
        }
    }
    *wpb = w;
    *smem = per_warp * w;
    return (int)((P + w - 1) / w);
}

// ---------------------------------------------------------------------------
// selection / decode epilogue
// ---------------------------------------------------------------------------
IL_HD size_t sel_warp_bytes(int n_r, int n_t, bool with_g) {
    const size_t N = 2 * (size_t)n_t;
    const size_t bytes = sizeof(cplx) * ((size_t)n_r * n_t + n_r) + (with_g ? 8 * (N * N + N) : 0);
    return (bytes + 15) / 16 * 16;
}

__global__ void k_select_decode(const double* __restrict__ Hg, const double* __restrict__ yg,
                                const double* __restrict__ Gg, const double* __restrict__ bg,
                                const double* __restrict__ offset, const int8_t* __restrict__ spins,
                                const uint8_t* __restrict__ diverged,
                                const double* __restrict__ energies, int64_t P, int n_r, int n_t,
                                int B, int Bs, Alphabet al, uint8_t* __restrict__ x_idx,
                                double* __restrict__ energy, int8_t* __restrict__ source,
                                int32_t* __restrict__ anneal_index,
                                int32_t* __restrict__ diverged_count) {
    extern __shared__ __align__(16) char smem_raw[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t prob = (int64_t)blockIdx.x * (blockDim.x >> 5) + warp;
    if (prob >= P) return;
    const int N = 2 * n_t, S = 2 * N + 1;
    // per-warp slice: H, y, then (only without precomputed energies) G, b
    const size_t per_warp = sel_warp_bytes(n_r, n_t, energies == nullptr);
    char* base = smem_raw + warp * per_warp;
    cplx* H = reinterpret_cast<cplx*>(base);
    cplx* y = H + n_r * n_t;
    double* G = reinterpret_cast<double*>(y + n_r);
    double* b = G + N * N;
    // H, y (and G, b when the anneal kernel did not supply energies) arrive by
    // 1-D TMA bulk copies issued by one lane: the warp's loads are in flight
    // while it reads the energies and flags (every size is a multiple of 16 B)
    __shared__ __align__(8) uint64_t bars[8];
    uint64_t* bar = &bars[warp];
    if (lane == 0) {
        mbar_init(bar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        const uint32_t hb = (uint32_t)(n_r * n_t * 16), yb = (uint32_t)(n_r * 16);
        const uint32_t gb = energies ? 0u : (uint32_t)(N * N * 8), bb = energies ? 0u : (uint32_t)(N * 8);
        mbar_expect_tx(bar, hb + yb + gb + bb);
        tma_bulk_g2s(H, Hg + prob * (int64_t)n_r * n_t * 2, hb, bar);
        tma_bulk_g2s(y, yg + prob * (int64_t)n_r * 2, yb, bar);
        if (!energies) {
            tma_bulk_g2s(G, Gg + prob * (int64_t)N * N, gb, bar);
            tma_bulk_g2s(b, bg + prob * (int64_t)N, bb, bar);
        }
    }
    __syncwarp();
    // with precomputed energies the selection needs H, y only for the decoded
    // residual: the argmin runs while the bulk copies are in flight
    const double e_guess_pre = energy[prob], off_pre = offset[prob];
    if (!energies) mbar_wait(bar, 0);
    double gsum = 0.0;
    if (!energies)
        for (int i = 0; i < N; ++i) gsum += G[i * N + i];

    // energies: lane = anneal, E = u'Gu - 2 tr G + 2 s_aux b'u  (solver.py:171-175)
    double best_e = INFINITY;
    int best_i = -1, ndiv = 0;
    // B anneals per problem in rows of stride Bs >= B (the fast kernel pads
    // B to a multiple of 16; padded anneals never enter the selection)
    const int8_t* sp0 = spins + prob * (int64_t)Bs * S;
    for (int a0 = 0; a0 < B; a0 += 32) {
        const int a = a0 + lane;
        double ea = INFINITY;
        if (a < B) {
            const bool dv = diverged[prob * Bs + a] != 0;
            ndiv += dv;
            if (!dv && energies) {
                ea = energies[prob * Bs + a];
            } else if (!dv) {
                const int8_t* s = sp0 + (int64_t)a * S;
                double quad = 0.0, lin = 0.0;
                for (int i = 0; i < N; ++i) {
                    const double ui = (double)(s[i] + s[N + i]);
                    if (ui == 0.0) continue;
                    double gu = 0.0;
                    for (int j = 0; j < N; ++j) gu += G[i * N + j] * (double)(s[j] + s[N + j]);
                    quad += ui * gu;
                    lin += b[i] * ui;
                }
                ea = (quad - 2.0 * gsum) + 2.0 * (double)s[2 * N] * lin;
            }
        }
        if (ea < best_e) {  // strict: earlier (lower) index wins ties
            best_e = ea;
            best_i = a;
        }
    }
    // warp argmin, ties -> lowest anneal index
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const double oe = __shfl_xor_sync(kFull, best_e, o);
        const int oi = __shfl_xor_sync(kFull, best_i, o);
        if (oe < best_e || (oe == best_e && oi >= 0 && (best_i < 0 || oi < best_i))) {
            best_e = oe;
            best_i = oi;
        }
    }
    ndiv = __reduce_add_sync(kFull, ndiv);
    if (diverged_count && lane == 0) diverged_count[prob] = ndiv;
    if (!(best_e < INFINITY)) best_i = -1;
    if (energies) mbar_wait(bar, 0);

    uint8_t* idx = x_idx + prob * 2 * n_t;
    const double e_guess = e_guess_pre;
    bool take = false;
    double e_dec = 0.0;
    __shared__ uint8_t cand_all[8][128];
    __shared__ cplx xs_all[8][64];
    uint8_t* cand = cand_all[warp];
    if (best_i >= 0 && !(best_e + off_pre > e_guess)) {
        const int8_t* s = sp0 + (int64_t)best_i * S;
        const int aux = s[2 * N];
        for (int k = lane; k < N; k += 32) {
            const int u = s[k] + s[N + k];  // -2, 0, 2
            const int user = k % n_t, part = k / n_t;  // k < n_t: real part
            int v = (int)idx[2 * user + part] + aux * (u / 2);
            v = v < 0 ? 0 : (v > al.m - 1 ? al.m - 1 : v);
            cand[2 * user + part] = (uint8_t)v;
        }
        __syncwarp();
        // residual of the decoded vector (linear.py:44-47)
        cplx* xs = xs_all[warp];
        for (int j = lane; j < n_t; j += 32) xs[j] = {al.levels[cand[2 * j]], al.levels[cand[2 * j + 1]]};
        __syncwarp();
        double acc = 0.0;
        for (int k = lane; k < n_r; k += 32)
            acc = __dadd_rn(acc, abs2_rn(resid_row(H + k * n_t, xs, n_t, y[k])));
        e_dec = warp_sum(acc);
        take = e_dec < e_guess;
    }
    if (take) {
        for (int k = lane; k < 2 * n_t; k += 32) idx[k] = cand[k];
        if (lane == 0) {
            energy[prob] = e_dec;
            if (source) source[prob] = IL_SRC_ANNEAL;
            if (anneal_index) anneal_index[prob] = best_i;
        }
    } else if (lane == 0) {
        if (source && source[prob] != IL_SRC_FAILED) source[prob] = IL_SRC_GUESS;
        if (anneal_index) anneal_index[prob] = -1;
    }
}

// ---------------------------------------------------------------------------
// ZF / VPP front-end (precoder.py:54-60, 93-125)
// ---------------------------------------------------------------------------
#ifndef IL_VPP_GROUPS  // 8-lane groups (4 problems per warp) for n_u, n_ant <= 8
#define IL_VPP_GROUPS 1
#endif
// GS lanes per problem (32: one warp; 8: four problems per warp when n_u and
// n_ant are <= 8); every element is computed by one lane with the same
// sequence of operations whichever GS, and the group sums add the same
// nonzero terms in the same tree order, so the outputs are bit-identical.
template <int GS>
__global__ void k_zf_vpp_front(const double* __restrict__ Hg, const double* __restrict__ ug,
                               int64_t P, int n_u, int n_ant, double tau, double* __restrict__ Wg,
                               double* __restrict__ ytg, double* __restrict__ Hpg,
                               double* __restrict__ base_energy, int8_t* __restrict__ status) {
    extern __shared__ __align__(16) char smem_raw[];
    const int lane = threadIdx.x & (GS - 1), warp = threadIdx.x / GS;  // group lane, group
    const unsigned mask = GS == 32 ? kFull : (((1u << GS) - 1u) << ((threadIdx.x & 31) & ~(GS - 1)));
    const int64_t prob = (int64_t)blockIdx.x * (blockDim.x / GS) + warp;
    if (prob >= P) return;  // whole groups exit together
    const size_t per_warp = sizeof(cplx) * ((size_t)n_u * n_ant * 2 + (size_t)n_u * n_u + n_u);
    cplx* H = reinterpret_cast<cplx*>(smem_raw + warp * per_warp);  // [n_u x n_ant]
    cplx* X = H + n_u * n_ant;                                      // [n_u x n_ant]
    cplx* L = X + n_u * n_ant;                                      // [n_u x n_u]
    cplx* u = L + n_u * n_u;
    const cplx* Hp = reinterpret_cast<const cplx*>(Hg) + prob * (int64_t)n_u * n_ant;
    for (int i = lane; i < n_u * n_ant; i += GS) H[i] = X[i] = Hp[i];
    for (int i = lane; i < n_u; i += GS) u[i] = reinterpret_cast<const cplx*>(ug)[prob * n_u + i];
    __syncwarp(mask);
    // A = H H^H  (row i of H against row j)
    for (int idx = lane; idx < n_u * n_u; idx += GS) {
        const int i = idx / n_u, j = idx % n_u;
        if (i > j) continue;
        double re = 0.0, im = 0.0;
        for (int k = 0; k < n_ant; ++k) {
            const cplx a = H[i * n_ant + k], bb = H[j * n_ant + k];
            re += a.re * bb.re + a.im * bb.im;
            im += a.im * bb.re - a.re * bb.im;
        }
        if (i == j) im = 0.0;
        L[i * n_u + j] = {re, im};
        L[j * n_u + i] = {re, -im};
    }
    __syncwarp(mask);
    __shared__ double invd_all[32][32];
    double* invd = invd_all[warp];
    const bool ok = GS == 32 ? cholesky_lower(L, n_u, invd, lane)
                             : cholesky_lower_g(L, n_u, invd, lane, mask);
    if (lane == 0 && status) status[prob] = ok ? 0 : -1;
    // X = A^-1 H, one column per lane
    for (int col = lane; col < n_ant; col += GS) {
        if (!ok) break;
        for (int k = 0; k < n_u; ++k) {
            const double lkk = L[k * n_u + k].re;
            cplx acc = X[k * n_ant + col];
            for (int j = 0; j < k; ++j) acc = csub(acc, cmul(L[k * n_u + j], X[j * n_ant + col]));
            X[k * n_ant + col] = {acc.re / lkk, acc.im / lkk};
        }
        for (int k = n_u - 1; k >= 0; --k) {
            const double lkk = L[k * n_u + k].re;
            cplx acc = X[k * n_ant + col];
            for (int j = k + 1; j < n_u; ++j) acc = csub(acc, cmulc(L[j * n_u + k], X[j * n_ant + col]));
            X[k * n_ant + col] = {acc.re / lkk, acc.im / lkk};
        }
    }
    __syncwarp(mask);
    // W = X^H [n_ant x n_u]; y_t = W u; H_p = -tau/2 W
    cplx* W = reinterpret_cast<cplx*>(Wg) + prob * (int64_t)n_ant * n_u;
    cplx* Hq = reinterpret_cast<cplx*>(Hpg) + prob * (int64_t)n_ant * n_u;
    const double ht = -tau / 2.0;
    for (int idx = lane; idx < n_ant * n_u; idx += GS) {
        const int a = idx / n_u, i = idx % n_u;
        const cplx xv = X[i * n_ant + a];
        const cplx wv = {xv.re, -xv.im};
        W[idx] = wv;
        Hq[idx] = {ht * wv.re, ht * wv.im};
    }
    double acc = 0.0;
    cplx* yt = reinterpret_cast<cplx*>(ytg) + prob * (int64_t)n_ant;
    for (int a = lane; a < n_ant; a += GS) {
        cplx s = {0.0, 0.0};
        for (int i = 0; i < n_u; ++i) {
            const cplx xv = X[i * n_ant + a];
            s = cadd(s, cmul(cplx{xv.re, -xv.im}, u[i]));
        }
        yt[a] = s;
        acc += cabs2(s);
    }
    if constexpr (GS == 32) {
        acc = warp_sum(acc);
    } else {  // the nonzero levels of warp_sum's tree (lanes >= GS hold 0)
#pragma unroll
        for (int o = GS / 2; o > 0; o >>= 1) acc = __dadd_rn(acc, __shfl_xor_sync(mask, acc, o, GS));
    }
    if (lane == 0) base_energy[prob] = acc;
}

// VPP epilogue (precoder.py:126-146).
__global__ void k_vpp_post(const double* __restrict__ Wg, const double* __restrict__ ug,
                           const double* __restrict__ ytg, const double* __restrict__ base_energy,
                           const uint8_t* __restrict__ vidx, int64_t P, int n_u, int n_ant,
                           int reach, double tau, double sqrtP, double* __restrict__ xg,
                           double* __restrict__ vg, double* __restrict__ powg) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t prob = (int64_t)blockIdx.x * (blockDim.x >> 5) + warp;
    if (prob >= P) return;
    const cplx* W = reinterpret_cast<const cplx*>(Wg) + prob * (int64_t)n_ant * n_u;
    const cplx* u = reinterpret_cast<const cplx*>(ug) + prob * (int64_t)n_u;
    const cplx* yt = reinterpret_cast<const cplx*>(ytg) + prob * (int64_t)n_ant;
    const uint8_t* vi = vidx + prob * 2 * n_u;
    cplx* v = reinterpret_cast<cplx*>(vg) + prob * (int64_t)n_u;
    cplx* x = reinterpret_cast<cplx*>(xg) + prob * (int64_t)n_ant;
    // perturbed = W (u + tau v), v = vhat / 2, vhat = 4 (idx - reach)
    double acc = 0.0;
    cplx pk[2] = {{0, 0}, {0, 0}};
    for (int a = lane, q = 0; a < n_ant; a += 32, ++q) {
        cplx s = {0.0, 0.0};
        for (int i = 0; i < n_u; ++i) {
            const cplx vv = {4.0 * (double)((int)vi[2 * i] - reach) / 2.0,
                             4.0 * (double)((int)vi[2 * i + 1] - reach) / 2.0};
            const cplx t = {u[i].re + tau * vv.re, u[i].im + tau * vv.im};
            s = cadd(s, cmul(W[a * n_u + i], t));
        }
        pk[q] = s;
        acc += cabs2(s);
    }
    double power = warp_sum(acc);
    const double base = base_energy[prob];
    const bool reject = power > base;
    if (reject) power = base;
    for (int i = lane; i < n_u; i += 32) {
        v[i] = reject ? cplx{0.0, 0.0}
                      : cplx{4.0 * (double)((int)vi[2 * i] - reach) / 2.0,
                             4.0 * (double)((int)vi[2 * i + 1] - reach) / 2.0};
    }
    const double nrm = sqrt(power);
    for (int a = lane, q = 0; a < n_ant; a += 32, ++q) {
        const cplx pa = reject ? yt[a] : pk[q];
        x[a] = nrm == 0.0 ? cplx{0.0, 0.0} : cplx{sqrtP * pa.re / nrm, sqrtP * pa.im / nrm};
    }
    if (lane == 0) powg[prob] = power;
}

__global__ void k_base_seeds(const uint64_t* __restrict__ seed, int64_t P, uint64_t k1, uint64_t k2,
                             uint64_t* __restrict__ out) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < P) out[i] = derive_seed3(seed[i], k1, k2);
}

// ||y - Hx||^2 per problem for arbitrary complex x (linear.py:44-47), in the
// library's one residual arithmetic (resid_row + 32-lane warp_sum).
__global__ void k_residual(const double* __restrict__ Hg, const double* __restrict__ yg,
                           const double* __restrict__ xg, int64_t P, int n_r, int n_t,
                           double* __restrict__ out) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t prob = (int64_t)blockIdx.x * (blockDim.x >> 5) + warp;
    if (prob >= P) return;
    const cplx* H = reinterpret_cast<const cplx*>(Hg) + prob * (int64_t)n_r * n_t;
    const cplx* y = reinterpret_cast<const cplx*>(yg) + prob * (int64_t)n_r;
    const cplx* x = reinterpret_cast<const cplx*>(xg) + prob * (int64_t)n_t;
    double acc = 0.0;
    for (int k = lane; k < n_r; k += 32) acc = __dadd_rn(acc, abs2_rn(resid_row(H + k * n_t, x, n_t, y[k])));
    acc = warp_sum(acc);
    if (lane == 0) out[prob] = acc;
}

__global__ void k_add_i32(const int32_t* __restrict__ a, int64_t n, int32_t* __restrict__ acc) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) acc[i] += a[i];
}

}  // namespace

int launch_residual(const double* H, const double* y, const double* x, int64_t P, int n_r, int n_t,
                    double* out, cudaStream_t st) {
    if (P == 0) return IL_OK;
    IL_LAUNCH(kProfOther, st, k_residual<<<(unsigned)((P + 3) / 4), 128, 0, st>>>(H, y, x, P, n_r, n_t, out););
    IL_CHECK_CUDA(cudaGetLastError());
    return IL_OK;
}

int launch_add_i32(const int32_t* a, int64_t n, int32_t* acc, cudaStream_t st) {
    if (n == 0) return IL_OK;
    IL_LAUNCH(kProfOther, st, k_add_i32<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(a, n, acc););
    IL_CHECK_CUDA(cudaGetLastError());
    return IL_OK;
}

// ---------------------------------------------------------------------------
// launchers
// ---------------------------------------------------------------------------
static int set_smem(const void* fn, size_t smem) {
    IL_REQUIRE(smem <= 227 * 1024, "per-problem matrices too large for shared memory (%zu B)", smem);
    IL_CHECK_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    return IL_OK;
}

int launch_mmse(const double* H, const double* y, const double* noise_var, int64_t P, int n_r,
                int n_t, const Alphabet& al, uint8_t* x_idx, double* energy, int8_t* status,
                cudaStream_t st) {
    if (P == 0) return IL_OK;
    IsingOut o{};
    if (front_rows_supported(n_r, n_t))
        return launch_front_rows(true, false, H, y, noise_var, P, n_r, n_t, al, x_idx, energy,
                                 status, o, st);
    int wpb;
    size_t smem;
    const int blocks = front_blocks(P, FrontSmem::bytes(n_r, n_t), &wpb, &smem);
    int rc = set_smem((const void*)k_front<true, false>, smem);
    if (rc) return rc;
    IL_LAUNCH(kProfFront, st, k_front<true, false><<<blocks, 32 * wpb, smem, st>>>(H, y, noise_var, P, n_r, n_t, al, x_idx,
                                                          energy, status, o););
    IL_CHECK_CUDA(cudaGetLastError());
    return IL_OK;
}

int launch_build_ising(const double* H, const double* y, const uint8_t* guess_idx, int64_t P,
                       int n_r, int n_t, const Alphabet& al, double* G, double* g_diag,
                       double* b, double* offset, double* eps_scale, double* eps_out,
                       double eps_gain, double fixed_eps, cudaStream_t st, double* gstats) {
    if (P == 0) return IL_OK;
    IsingOut o{G, g_diag, b, offset, eps_scale, eps_out, eps_gain, fixed_eps};
    IL_REQUIRE(!gstats || front_rows_supported(n_r, n_t), "gstats come from the row front end only");
    o.gstats = gstats;
    if (front_rows_supported(n_r, n_t))
        return launch_front_rows(false, true, H, y, nullptr, P, n_r, n_t, al,
                                 const_cast<uint8_t*>(guess_idx), nullptr, nullptr, o, st);
    int wpb;
    size_t smem;
    const int blocks = front_blocks(P, FrontSmem::bytes(n_r, n_t), &wpb, &smem);
    int rc = set_smem((const void*)k_front<false, true>, smem);
    if (rc) return rc;
    IL_LAUNCH(kProfFront, st, k_front<false, true><<<blocks, 32 * wpb, smem, st>>>(H, y, nullptr, P, n_r, n_t, al,
                                                          const_cast<uint8_t*>(guess_idx),
                                                          nullptr, nullptr, o););
    IL_CHECK_CUDA(cudaGetLastError());
    return IL_OK;
}

int launch_mmse_ising(const double* H, const double* y, const double* noise_var, int64_t P,
                      int n_r, int n_t, const Alphabet& al, uint8_t* x_idx, double* energy,
                      int8_t* status, double* G, double* g_diag, double* b, double* offset,
                      double* eps_out, double eps_gain, double fixed_eps, cudaStream_t st,
                      double* gstats) {
    if (P == 0) return IL_OK;
    IsingOut o{G, g_diag, b, offset, nullptr, eps_out, eps_gain, fixed_eps};
    IL_REQUIRE(!gstats || front_rows_supported(n_r, n_t), "gstats come from the row front end only");
    o.gstats = gstats;
    if (front_rows_supported(n_r, n_t))
        return launch_front_rows(true, true, H, y, noise_var, P, n_r, n_t, al, x_idx, energy,
                                 status, o, st);
    int wpb;
    size_t smem;
    const int blocks = front_blocks(P, FrontSmem::bytes(n_r, n_t), &wpb, &smem);
    int rc = set_smem((const void*)k_front<true, true>, smem);
    if (rc) return rc;
    IL_LAUNCH(kProfFront, st, k_front<true, true><<<blocks, 32 * wpb, smem, st>>>(H, y, noise_var, P, n_r, n_t, al, x_idx,
                                                         energy, status, o););
    IL_CHECK_CUDA(cudaGetLastError());
    return IL_OK;
}

int launch_select_decode(const double* H, const double* y, const double* G, const double* b,
                         const double* offset, const int8_t* spins, const uint8_t* diverged,
                         const double* energies, int64_t P, int n_r, int n_t, int B, int Bs,
                         const Alphabet& al, uint8_t* x_idx_io, double* energy_io,
                         int8_t* source, int32_t* anneal_index, int32_t* diverged_count,
                         cudaStream_t st) {
    if (P == 0) return IL_OK;
    const int N = 2 * n_t;
    IL_REQUIRE(2 * n_t <= 128, "n_t too large");
    // H, y (and G, b) arrive by 1-D bulk copies: 16-byte aligned sources
    IL_REQUIRE((((uintptr_t)H | (uintptr_t)y | (uintptr_t)G | (uintptr_t)b) & 15u) == 0,
               "H and y must be 16-byte aligned (complex128 device arrays)");
    const size_t per_warp = sel_warp_bytes(n_r, n_t, energies == nullptr);
    int wpb = (int)((200 * 1024) / per_warp);
    wpb = wpb < 1 ? 1 : (wpb > 8 ? 8 : wpb);
    const size_t smem = per_warp * wpb;
    int rc = set_smem((const void*)k_select_decode, smem);
    if (rc) return rc;
    const int blocks = (int)((P + wpb - 1) / wpb);
    IL_LAUNCH(kProfSelect, st, k_select_decode<<<blocks, 32 * wpb, smem, st>>>(H, y, G, b, offset, spins, diverged, energies, P, n_r,
                                                    n_t, B, Bs, al, x_idx_io, energy_io, source,
                                                    anneal_index, diverged_count););
    IL_CHECK_CUDA(cudaGetLastError());
    return IL_OK;
}

int launch_zf_vpp_front(const double* H, const double* u, int64_t P, int n_u, int n_ant,
                        double tau, double* W, double* y_t, double* H_p, double* base_energy,
                        int8_t* status, cudaStream_t st) {
    if (P == 0) return IL_OK;
    const size_t per_warp = sizeof(cplx) * ((size_t)n_u * n_ant * 2 + (size_t)n_u * n_u + n_u);
    if (n_u <= 8 && n_ant <= 8 && IL_VPP_GROUPS) {  // four problems per warp, 16 per block
        constexpr int GS = 8, kGroups = 16;
        const size_t smem = per_warp * kGroups;
        int rc = set_smem((const void*)k_zf_vpp_front<GS>, smem);
        if (rc) return rc;
        const int blocks = (int)((P + kGroups - 1) / kGroups);
        IL_LAUNCH(kProfFront, st, k_zf_vpp_front<GS><<<blocks, GS * kGroups, smem, st>>>(H, u, P, n_u, n_ant, tau, W, y_t, H_p,
                                                       base_energy, status););
        IL_CHECK_CUDA(cudaGetLastError());
        return IL_OK;
    }
    int wpb = (int)((200 * 1024) / per_warp);
    wpb = wpb < 1 ? 1 : (wpb > 4 ? 4 : wpb);
    const size_t smem = per_warp * wpb;
    int rc = set_smem((const void*)k_zf_vpp_front<32>, smem);
    if (rc) return rc;
    const int blocks = (int)((P + wpb - 1) / wpb);
    IL_LAUNCH(kProfFront, st, k_zf_vpp_front<32><<<blocks, 32 * wpb, smem, st>>>(H, u, P, n_u, n_ant, tau, W, y_t, H_p,
                                                   base_energy, status););
    IL_CHECK_CUDA(cudaGetLastError());
    return IL_OK;
}

int launch_vpp_post(const double* W, const double* u, const double* y_t, const double* base_energy,
                    const uint8_t* vidx, int64_t P, int n_u, int n_ant, int reach, double tau,
                    double power, double* x, double* v, double* unnorm_power, cudaStream_t st) {
    if (P == 0) return IL_OK;
    IL_REQUIRE(n_ant <= 64, "n_ant > 64 not supported");
    const int wpb = 4;
    const int blocks = (int)((P + wpb - 1) / wpb);
    IL_LAUNCH(kProfOther, st, k_vpp_post<<<blocks, 32 * wpb, 0, st>>>(W, u, y_t, base_energy, vidx, P, n_u, n_ant, reach,
                                            tau, sqrt(power), x, v, unnorm_power););
    IL_CHECK_CUDA(cudaGetLastError());
    return IL_OK;
}

int launch_base_seeds(const uint64_t* seed, int64_t P, uint64_t k1, uint64_t k2,
                      uint64_t* base_out, cudaStream_t st) {
    if (P == 0) return IL_OK;
    IL_LAUNCH(kProfOther, st, k_base_seeds<<<(unsigned)((P + 255) / 256), 256, 0, st>>>(seed, P, k1, k2, base_out););
    IL_CHECK_CUDA(cudaGetLastError());
    return IL_OK;
}

}  // namespace il

// ---------------------------------------------------------------------------
// Gray demapper (channel.py:160-180): per PAM dimension label = idx ^ (idx >> 1)
// ---------------------------------------------------------------------------
namespace il {
namespace {
__global__ void k_gray_demap(const uint8_t* __restrict__ x_idx, int64_t n_dims, int bpd,
                             uint8_t* __restrict__ bits) {
    const int64_t d = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (d >= n_dims) return;
    const unsigned k = x_idx[d];
    const unsigned gl = k ^ (k >> 1);
    for (int q = 0; q < bpd; ++q) bits[d * bpd + q] = (uint8_t)((gl >> (bpd - 1 - q)) & 1u);
}
}  // namespace

int launch_gray_demap(const uint8_t* x_idx, int64_t n_sym, int bits_per_dim, uint8_t* bits,
                      cudaStream_t st) {
    IL_REQUIRE(bits_per_dim >= 1 && bits_per_dim <= 8, "bits_per_dim must be in [1, 8]");
    const int64_t n = 2 * n_sym;
    if (n == 0) return IL_OK;
    IL_LAUNCH(kProfOther, st, k_gray_demap<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(x_idx, n, bits_per_dim, bits););
    IL_CHECK_CUDA(cudaGetLastError());
    return IL_OK;
}
}  // namespace il
