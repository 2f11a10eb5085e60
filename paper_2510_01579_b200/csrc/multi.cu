// MMGaP-E: batched MMSE-SIC and the multi-chain, multi-stage detector.
//
//   k_mmse_sic          linear.py:78-106   ordered MMSE-SIC hard decision
//   detect_cim_multi    detector.py:85-134 two guess chains (MMSE, MMSE-SIC) x
//                                          n_stages of _improve_guess, best of all
//
// k_mmse_sic follows the register-resident layout of front_rows.cu: a group
// of GS lanes owns one resource element, lane r owns row r.  Each SIC round
// forms the regularised Gram matrix of the remaining users (removed users
// become identity rows/columns, which leaves the remaining block's inverse
// unchanged), inverts it in place by Gauss-Jordan (no pivoting: the matrix
// is Hermitian positive definite; a pivot <= 0 is cho_factor's failure),
// takes x_soft = A^-1 Hs^H y_res and decides the remaining user with the
// smallest diag(A^-1) (first minimum, np.argmin), then cancels it from y_res.
#include "il_group.cuh"
#include "il_internal.cuh"

namespace il {
namespace {

constexpr int kSicThreads = 128;

IL_HD size_t sic_group_cplx(int n_r, int n, int GS) {
    // H, y, y_res, Gram, pivot row, z broadcast
    return (size_t)n_r * n + 2 * (size_t)n_r + (size_t)n * n + 2 * (size_t)GS + 2;
}

template <int GS>
__global__ void __launch_bounds__(kSicThreads, GS <= 16 ? 4 : 1)
k_mmse_sic(const double* __restrict__ Hg, const double* __restrict__ yg,
           const double* __restrict__ s2g, int64_t P, int n_r, int n, Alphabet al,
           uint8_t* __restrict__ x_idx, double* __restrict__ energy, int8_t* __restrict__ status) {
    extern __shared__ __align__(16) cplx smem_c[];
    const Grp<GS> g;
    const int r = g.r;
    const int grp = threadIdx.x / GS;
    const int64_t prob = (int64_t)blockIdx.x * (kSicThreads / GS) + grp;
    if (prob >= P) return;
    cplx* H = smem_c + grp * sic_group_cplx(n_r, n, GS);
    cplx* y = H + n_r * n;
    cplx* yres = y + n_r;
    cplx* Ag = yres + n_r;      // Gram H^H H [n][n]
    cplx* rowb = Ag + n * n;    // pivot row broadcast [GS]
    cplx* zb = rowb + GS;       // z broadcast [GS]
    cplx* symb = zb + GS;       // decided symbol broadcast [1]
    {
        const cplx* Hp = reinterpret_cast<const cplx*>(Hg) + prob * (int64_t)n_r * n;
        for (int i = r; i < n_r * n; i += GS) H[i] = Hp[i];
        const cplx* yp = reinterpret_cast<const cplx*>(yg) + prob * (int64_t)n_r;
        for (int i = r; i < n_r; i += GS) y[i] = yres[i] = yp[i];
    }
    g.sync();
    // Gram rows (Im part as two sums: exactly Hermitian, real diagonal)
    if (r < n) {
        double re[GS], i1[GS], i2[GS];
#pragma unroll
        for (int j = 0; j < GS; ++j) re[j] = i1[j] = i2[j] = 0.0;
        for (int k = 0; k < n_r; ++k) {
            const cplx hr = H[k * n + r];
#pragma unroll
            for (int j = 0; j < GS; ++j) {
                if (j < n) {
                    const cplx hj = H[k * n + j];
                    re[j] = fma(hr.re, hj.re, fma(hr.im, hj.im, re[j]));
                    i1[j] = fma(hr.re, hj.im, i1[j]);
                    i2[j] = fma(hr.im, hj.re, i2[j]);
                }
            }
        }
#pragma unroll
        for (int j = 0; j < GS; ++j)
            if (j < n) Ag[r * n + j] = {re[j], i1[j] - i2[j]};
    }
    g.sync();
    const double rho = s2g[prob];
    uint8_t* idx = x_idx + prob * 2 * n;
    uint32_t removed = 0;
    bool ok = true;
#pragma unroll 1
    for (int round = 0; round < n; ++round) {
        const bool mine = r < n && !((removed >> r) & 1u);
        cplx A[GS];
#pragma unroll
        for (int j = 0; j < GS; ++j) {
            const bool live = mine && j < n && !((removed >> j) & 1u);
            A[j] = live ? Ag[r * n + j] : cplx{0.0, 0.0};
            if (j == r) A[j] = mine ? cplx{A[j].re + rho, A[j].im} : cplx{1.0, 0.0};
        }
        cplx zr = {0.0, 0.0};
        if (mine) {
            for (int k = 0; k < n_r; ++k) {
                const cplx h = H[k * n + r], v = yres[k];
                zr.re = fma(h.re, v.re, fma(h.im, v.im, zr.re));
                zr.im = fma(h.re, v.im, fma(-h.im, v.re, zr.im));
            }
        }
        // in-place Gauss-Jordan inversion
#pragma unroll
        for (int k = 0; k < GS; ++k) {
            if (k >= n) break;
            if (r == k) {
                const double p = A[k].re;
                ok = ok && (p > 0.0);
                const double inv = 1.0 / p;
#pragma unroll
                for (int j = 0; j < GS; ++j)
                    rowb[j] = (j == k) ? cplx{inv, 0.0} : cplx{A[j].re * inv, A[j].im * inv};
            }
            g.sync();
            if (r == k) {
#pragma unroll
                for (int j = 0; j < GS; ++j) A[j] = rowb[j];
            } else {
                const cplx f = A[k];
                const double inv = rowb[k].re;
#pragma unroll
                for (int j = 0; j < GS; ++j)
                    if (j != k) A[j] = csub(A[j], cmul(f, rowb[j]));
                A[k] = {-f.re * inv, -f.im * inv};
            }
            g.sync();
        }
        zb[r] = zr;
        g.sync();
        cplx xs = {0.0, 0.0};
        double dr = 0.0;
#pragma unroll
        for (int j = 0; j < GS; ++j) {
            xs = cadd(xs, cmul(A[j], zb[j]));
            if (j == r) dr = A[j].re;
        }
        // argmin of diag(A^-1) over the remaining users, first minimum
        double bv = mine ? dr : INFINITY;
        int bi = mine ? r : GS;
#pragma unroll
        for (int o = GS / 2; o > 0; o >>= 1) {
            const double ov = __shfl_xor_sync(g.mask, bv, o, GS);
            const int oi = __shfl_xor_sync(g.mask, bi, o, GS);
            if (ov < bv || (ov == bv && oi < bi)) {
                bv = ov;
                bi = oi;
            }
        }
        if (r == bi) {
            const int kr = level_index(xs.re, al), ki = level_index(xs.im, al);
            idx[2 * r] = (uint8_t)kr;
            idx[2 * r + 1] = (uint8_t)ki;
            symb[0] = {al.levels[kr], al.levels[ki]};
        }
        g.sync();
        const cplx sym = symb[0];
        for (int k = r; k < n_r; k += GS) {  // y_res -= H[:, user] * sym
            const cplx h = H[k * n + bi];
            const cplx t = {__dsub_rn(__dmul_rn(h.re, sym.re), __dmul_rn(h.im, sym.im)),
                            __dadd_rn(__dmul_rn(h.re, sym.im), __dmul_rn(h.im, sym.re))};
            yres[k] = {__dsub_rn(yres[k].re, t.re), __dsub_rn(yres[k].im, t.im)};
        }
        removed |= 1u << bi;
        g.sync();
    }
    // residual of the decision (linear.py:44-47), same arithmetic as every
    // other energy in the library; the 32-lane summation tree is emulated
    cplx* xsym = rowb;
    if (r < n) xsym[r] = {al.levels[idx[2 * r]], al.levels[idx[2 * r + 1]]};
    g.sync();
    for (int k = r; k < n_r; k += GS) yres[k] = resid_row(H + k * n, xsym, n, y[k]);
    g.sync();
    double acc;
    {
        double a[32 / GS];
#pragma unroll
        for (int q = 0; q < 32 / GS; ++q) {
            a[q] = 0.0;
            for (int k = r + q * GS; k < n_r; k += 32) a[q] = __dadd_rn(a[q], abs2_rn(yres[k]));
        }
        if (GS == 32) acc = a[0];
        else if (GS == 16) acc = __dadd_rn(a[0], a[1]);
        else acc = __dadd_rn(__dadd_rn(a[0], a[2]), __dadd_rn(a[1], a[3]));
    }
    const double r2 = g.sum(acc);
    const bool all_ok = __all_sync(g.mask, ok);
    if (r == 0) {
        if (energy) energy[prob] = r2;
        if (status) status[prob] = all_ok ? 0 : -1;
    }
}

template <int GS>
int launch_sic_gs(const double* H, const double* y, const double* s2, int64_t P, int n_r, int n,
                  const Alphabet& al, uint8_t* x_idx, double* energy, int8_t* status,
                  cudaStream_t st) {
    const int groups = kSicThreads / GS;
    const size_t smem = sizeof(cplx) * sic_group_cplx(n_r, n, GS) * groups;
    IL_REQUIRE(smem <= 227 * 1024, "MMSE-SIC problem too large for shared memory");
    auto fn = k_mmse_sic<GS>;
    IL_CHECK_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    const int64_t blocks = (P + groups - 1) / groups;
    IL_LAUNCH(kProfFront, st,
              fn<<<(unsigned)blocks, kSicThreads, smem, st>>>(H, y, s2, P, n_r, n, al, x_idx,
                                                              energy, status););
    IL_CHECK_CUDA(cudaGetLastError());
    return IL_OK;
}

// ---- multi-chain bookkeeping (detector.py:110-134) --------------------------
// best <- first minimum-energy baseline
__global__ void k_multi_init(const uint8_t* __restrict__ bx, const double* __restrict__ be,
                             const int8_t* __restrict__ bst, const int32_t* __restrict__ codes,
                             int n_chains, int64_t P, int nx, uint8_t* __restrict__ x,
                             double* __restrict__ e, int8_t* __restrict__ src,
                             int32_t* __restrict__ aidx) {
    const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= P) return;
    int best = 0;
    bool failed = false;
    for (int c = 0; c < n_chains; ++c) {
        failed = failed || bst[c * P + p] != 0;
        if (be[c * P + p] < be[best * P + p]) best = c;
    }
    for (int k = 0; k < nx; ++k) x[p * nx + k] = bx[(best * P + p) * nx + k];
    e[p] = be[best * P + p];
    src[p] = failed ? IL_SRC_FAILED : (codes[best] == 0 ? IL_SRC_GUESS : IL_SRC_SIC);
    aidx[p] = -1;
}

// widx <- stage winner if the stage improved
__global__ void k_multi_stage(const int32_t* __restrict__ stage_ai, int64_t P,
                              int32_t* __restrict__ widx) {
    const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (p < P && stage_ai[p] >= 0) widx[p] = stage_ai[p];
}

// best <- chain result if strictly better
__global__ void k_multi_combine(const uint8_t* __restrict__ gx, const double* __restrict__ ge,
                                const int32_t* __restrict__ widx, int64_t P, int nx,
                                uint8_t* __restrict__ x, double* __restrict__ e,
                                int8_t* __restrict__ src, int32_t* __restrict__ aidx) {
    const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= P || !(ge[p] < e[p])) return;
    for (int k = 0; k < nx; ++k) x[p * nx + k] = gx[p * nx + k];
    e[p] = ge[p];
    if (src[p] != IL_SRC_FAILED) src[p] = IL_SRC_ANNEAL;
    aidx[p] = widx[p];
}

}  // namespace

int launch_mmse_sic(const double* H, const double* y, const double* noise_var, int64_t P, int n_r,
                    int n_t, const Alphabet& al, uint8_t* x_idx, double* energy, int8_t* status,
                    cudaStream_t st) {
    if (P == 0) return IL_OK;
    if (n_t <= 8) return launch_sic_gs<8>(H, y, noise_var, P, n_r, n_t, al, x_idx, energy, status, st);
    if (n_t <= 16) return launch_sic_gs<16>(H, y, noise_var, P, n_r, n_t, al, x_idx, energy, status, st);
    return launch_sic_gs<32>(H, y, noise_var, P, n_r, n_t, al, x_idx, energy, status, st);
}

int launch_multi_init(const uint8_t* bx, const double* be, const int8_t* bst,
                      const int32_t* codes, int n_chains, int64_t P, int nx, uint8_t* x,
                      double* e, int8_t* src, int32_t* aidx, cudaStream_t st) {
    if (P == 0) return IL_OK;
    IL_LAUNCH(kProfOther, st,
              k_multi_init<<<(unsigned)((P + 255) / 256), 256, 0, st>>>(bx, be, bst, codes, n_chains,
                                                                      P, nx, x, e, src, aidx););
    IL_CHECK_CUDA(cudaGetLastError());
    return IL_OK;
}

int launch_multi_stage(const int32_t* stage_ai, int64_t P, int32_t* widx, cudaStream_t st) {
    if (P == 0) return IL_OK;
    IL_LAUNCH(kProfOther, st,
              k_multi_stage<<<(unsigned)((P + 255) / 256), 256, 0, st>>>(stage_ai, P, widx););
    IL_CHECK_CUDA(cudaGetLastError());
    return IL_OK;
}

int launch_multi_combine(const uint8_t* gx, const double* ge, const int32_t* widx, int64_t P,
                         int nx, uint8_t* x, double* e, int8_t* src, int32_t* aidx,
                         cudaStream_t st) {
    if (P == 0) return IL_OK;
    IL_LAUNCH(kProfOther, st,
              k_multi_combine<<<(unsigned)((P + 255) / 256), 256, 0, st>>>(gx, ge, widx, P, nx, x, e,
                                                                         src, aidx););
    IL_CHECK_CUDA(cudaGetLastError());
    return IL_OK;
}

}  // namespace il
