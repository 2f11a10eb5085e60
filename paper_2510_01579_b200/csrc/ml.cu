// Exhaustive maximum-likelihood detection (linear.py:109-144) on the GPU:
// the SER floor the reference's sweeps report as detector "ml".
//
// One CTA per resource element.  Candidate k enumerates symbol indices with
// user 0 most significant (k = sum_j d_j M^(n_t-1-j), points[d] =
// pam[d / m] + i pam[d % m], channel.py:102); ties go to the smallest k, as
// the reference's chunked argmin does.  A thread owns a prefix (the symbols
// of users 0..n_t-2) and sweeps the last user's M symbols, so the residual of
// the prefix is formed once per M candidates; every candidate's energy is
// y - H_0 x_0 - ... - H_{n-1} x_{n-1} accumulated in user order with
// explicitly rounded operations, i.e. the same value whichever thread
// evaluates it.  The reference refuses search spaces above 24 bits.
#include "il_internal.cuh"

namespace il {
namespace {

constexpr int kMlThreads = 256;
constexpr int kMlMaxNr = 32;

IL_D cplx sub_mul(cplx r, cplx h, cplx x) {  // r - h x, each operation rounded
    const double pr = __dsub_rn(__dmul_rn(h.re, x.re), __dmul_rn(h.im, x.im));
    const double pi = __dadd_rn(__dmul_rn(h.re, x.im), __dmul_rn(h.im, x.re));
    return {__dsub_rn(r.re, pr), __dsub_rn(r.im, pi)};
}

__global__ void __launch_bounds__(kMlThreads)
k_ml(const double* __restrict__ Hg, const double* __restrict__ yg, int64_t P, int n_r, int n_t,
     Alphabet al, int64_t n_prefix, uint8_t* __restrict__ x_idx, double* __restrict__ energy) {
    extern __shared__ __align__(16) cplx sm[];
    const int64_t prob = blockIdx.x;
    if (prob >= P) return;
    const int m = al.m, M = m * m;
    cplx* H = sm;              // [n_r][n_t]
    cplx* y = H + n_r * n_t;   // [n_r]
    cplx* pts = y + n_r;       // [M]
    __shared__ double red_e[kMlThreads / 32];
    __shared__ long long red_k[kMlThreads / 32];
    const cplx* Hp = reinterpret_cast<const cplx*>(Hg) + prob * (int64_t)n_r * n_t;
    for (int i = threadIdx.x; i < n_r * n_t; i += kMlThreads) H[i] = Hp[i];
    for (int i = threadIdx.x; i < n_r; i += kMlThreads)
        y[i] = reinterpret_cast<const cplx*>(yg)[prob * n_r + i];
    for (int d = threadIdx.x; d < M; d += kMlThreads) pts[d] = {al.levels[d / m], al.levels[d % m]};
    __syncthreads();

    double best_e = INFINITY;
    long long best_k = -1;
    cplx r[kMlMaxNr];
    const int last = n_t - 1;
    for (int64_t pfx = threadIdx.x; pfx < n_prefix; pfx += kMlThreads) {
        // prefix residual y - sum_{j < last} H_j x_j (user 0 most significant)
#pragma unroll
        for (int i = 0; i < kMlMaxNr; ++i)
            if (i < n_r) r[i] = y[i];
        int64_t div = n_prefix;
        for (int j = 0; j < last; ++j) {
            div /= M;
            const cplx x = pts[(pfx / div) % M];
#pragma unroll
            for (int i = 0; i < kMlMaxNr; ++i)
                if (i < n_r) r[i] = sub_mul(r[i], H[i * n_t + j], x);
        }
        for (int d = 0; d < M; ++d) {
            const cplx x = pts[d];
            double e = 0.0;
#pragma unroll
            for (int i = 0; i < kMlMaxNr; ++i) {
                if (i < n_r) {
                    const cplx ri = sub_mul(r[i], H[i * n_t + last], x);
                    e = __dadd_rn(e, __fma_rn(ri.re, ri.re, __dmul_rn(ri.im, ri.im)));
                }
            }
            if (e < best_e) {  // candidates of a thread arrive in increasing k
                best_e = e;
                best_k = pfx * M + d;
            }
        }
    }
    // block argmin, ties -> smallest k
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const double oe = __shfl_xor_sync(0xffffffffu, best_e, o);
        const long long ok = __shfl_xor_sync(0xffffffffu, best_k, o);
        if (oe < best_e || (oe == best_e && ok >= 0 && (best_k < 0 || ok < best_k))) {
            best_e = oe;
            best_k = ok;
        }
    }
    if (lane == 0) {
        red_e[warp] = best_e;
        red_k[warp] = best_k;
    }
    __syncthreads();
    if (warp == 0) {
        best_e = lane < kMlThreads / 32 ? red_e[lane] : INFINITY;
        best_k = lane < kMlThreads / 32 ? red_k[lane] : -1;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const double oe = __shfl_xor_sync(0xffffffffu, best_e, o);
            const long long ok = __shfl_xor_sync(0xffffffffu, best_k, o);
            if (oe < best_e || (oe == best_e && ok >= 0 && (best_k < 0 || ok < best_k))) {
                best_e = oe;
                best_k = ok;
            }
        }
        // decode the winner and recompute its residual in the library's
        // common arithmetic (linear.py:144 recomputes residual_energy)
        cplx* xs = pts + M;  // n_t scratch after the points
        if (lane == 0) {
            long long k = best_k < 0 ? 0 : best_k;
            for (int j = n_t - 1; j >= 0; --j) {
                const int d = (int)(k % M);
                k /= M;
                x_idx[(prob * n_t + j) * 2] = (uint8_t)(d / m);
                x_idx[(prob * n_t + j) * 2 + 1] = (uint8_t)(d % m);
                xs[j] = pts[d];
            }
        }
        __syncwarp();
        double acc = 0.0;
        for (int k = lane; k < n_r; k += 32) acc = __dadd_rn(acc, abs2_rn(resid_row(H + k * n_t, xs, n_t, y[k])));
        acc = warp_sum(acc);
        if (lane == 0 && energy) energy[prob] = acc;
    }
}

// Max-log bit LLRs by the same exhaustive search (no reference: soft output is
// a non-goal of the reference, SPEC.md:153 -- the definition is the standard
// max-log one and is pinned only against the oracle's brute force):
//   LLR_b = (min_{x: b(x) = 1} ||y - Hx||^2 - min_{x: b(x) = 0} ||y - Hx||^2) / s2
// with bit b = (user j, re/im, Gray bit q MSB first) in the order of the Gray
// demapper (channel.py:160-180), so LLR_b > 0 favours bit 0.  A thread keeps
// the minima of the last user's bits per candidate and those of the prefix
// users once per prefix (the minimum over its M completions).
constexpr int kLlrMaxBits = 24, kLlrMaxLast = 16, kLlrMaxNr = 16;

__global__ void __launch_bounds__(kMlThreads)
k_ml_llr(const double* __restrict__ Hg, const double* __restrict__ yg,
         const double* __restrict__ noise_var, int64_t P, int n_r, int n_t, Alphabet al,
         int64_t n_prefix, int bpd, double* __restrict__ llr) {
    extern __shared__ __align__(16) cplx sm[];
    const int64_t prob = blockIdx.x;
    if (prob >= P) return;
    const int m = al.m, M = m * m, nb = 2 * bpd * n_t, nl = 2 * bpd, npre = nb - nl;
    cplx* H = sm;
    cplx* y = H + n_r * n_t;
    cplx* pts = y + n_r;
    __shared__ double red[2][kMlThreads / 32][kLlrMaxBits];
    const cplx* Hp = reinterpret_cast<const cplx*>(Hg) + prob * (int64_t)n_r * n_t;
    for (int i = threadIdx.x; i < n_r * n_t; i += kMlThreads) H[i] = Hp[i];
    for (int i = threadIdx.x; i < n_r; i += kMlThreads)
        y[i] = reinterpret_cast<const cplx*>(yg)[prob * n_r + i];
    for (int d = threadIdx.x; d < M; d += kMlThreads) pts[d] = {al.levels[d / m], al.levels[d % m]};
    __syncthreads();

    // Gray bits of symbol d as one 2 bpd-bit word: re label (high bits) then
    // im label, bit q of the symbol (MSB first) at 2 bpd - 1 - q
    auto sym_bits = [&](int d) -> int {
        const int ire = d / m, iim = d - ire * m;
        return ((ire ^ (ire >> 1)) << bpd) | (iim ^ (iim >> 1));
    };
    double mpre[2][kLlrMaxBits], mlast[2][kLlrMaxLast];
#pragma unroll
    for (int b = 0; b < kLlrMaxBits; ++b) mpre[0][b] = mpre[1][b] = INFINITY;
#pragma unroll
    for (int b = 0; b < kLlrMaxLast; ++b) mlast[0][b] = mlast[1][b] = INFINITY;
    cplx r[kLlrMaxNr];
    const int last = n_t - 1;
    for (int64_t pfx = threadIdx.x; pfx < n_prefix; pfx += kMlThreads) {
#pragma unroll
        for (int i = 0; i < kLlrMaxNr; ++i)
            if (i < n_r) r[i] = y[i];
        int64_t div = n_prefix;
        for (int j = 0; j < last; ++j) {
            div /= M;
            const cplx x = pts[(pfx / div) % M];
#pragma unroll
            for (int i = 0; i < kLlrMaxNr; ++i)
                if (i < n_r) r[i] = sub_mul(r[i], H[i * n_t + j], x);
        }
        double emin = INFINITY;
        for (int d = 0; d < M; ++d) {
            const cplx x = pts[d];
            double e = 0.0;
#pragma unroll
            for (int i = 0; i < kLlrMaxNr; ++i) {
                if (i < n_r) {
                    const cplx ri = sub_mul(r[i], H[i * n_t + last], x);
                    e = __dadd_rn(e, __fma_rn(ri.re, ri.re, __dmul_rn(ri.im, ri.im)));
                }
            }
            emin = fmin(emin, e);
            const int word = sym_bits(d);
#pragma unroll
            for (int q = 0; q < kLlrMaxLast; ++q) {
                if (q < nl) {
                    const int bit = (word >> (nl - 1 - q)) & 1;
                    mlast[0][q] = bit ? mlast[0][q] : fmin(mlast[0][q], e);
                    mlast[1][q] = bit ? fmin(mlast[1][q], e) : mlast[1][q];
                }
            }
        }
        // prefix users: the best completion of this prefix
#pragma unroll
        for (int b = 0; b < kLlrMaxBits; ++b) {
            if (b < npre) {
                const int j = b / nl, q = b % nl;
                int64_t dv = n_prefix;
                for (int k = 0; k <= j; ++k) dv /= M;
                const int bit = (sym_bits((int)((pfx / dv) % M)) >> (nl - 1 - q)) & 1;
                mpre[0][b] = bit ? mpre[0][b] : fmin(mpre[0][b], emin);
                mpre[1][b] = bit ? fmin(mpre[1][b], emin) : mpre[1][b];
            }
        }
    }
    // block minima per (bit value, position)
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int v = 0; v < 2; ++v) {
#pragma unroll
        for (int b = 0; b < kLlrMaxBits; ++b) {
            double x = b < npre ? mpre[v][b] : INFINITY;
            if (b >= npre && b - npre < kLlrMaxLast) {
#pragma unroll
                for (int q = 0; q < kLlrMaxLast; ++q)
                    if (q == b - npre) x = mlast[v][q];
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) x = fmin(x, __shfl_xor_sync(0xffffffffu, x, o));
            if (lane == 0) red[v][warp][b] = x;
        }
    }
    __syncthreads();
    if (threadIdx.x < nb) {
        const int b = threadIdx.x;
        double d0 = INFINITY, d1 = INFINITY;
        for (int w = 0; w < kMlThreads / 32; ++w) {
            d0 = fmin(d0, red[0][w][b]);
            d1 = fmin(d1, red[1][w][b]);
        }
        const double s2 = noise_var ? noise_var[prob] : 1.0;
        llr[prob * nb + b] = (d1 - d0) / s2;
    }
}

}  // namespace

int launch_ml(const double* H, const double* y, int64_t P, int n_r, int n_t, const Alphabet& al,
              uint8_t* x_idx, double* energy, cudaStream_t st) {
    if (P == 0) return IL_OK;
    IL_REQUIRE(n_r <= kMlMaxNr, "ML detection supports n_r <= %d", kMlMaxNr);
    const int M = al.m * al.m;
    int bits = 0;
    while ((1 << bits) < M) ++bits;
    IL_REQUIRE((int64_t)bits * n_t <= 24, "ML search space of %d bits exceeds the 24-bit guard",
               bits * n_t);
    int64_t n_prefix = 1;
    for (int j = 0; j < n_t - 1; ++j) n_prefix *= M;
    const size_t smem = sizeof(cplx) * ((size_t)n_r * n_t + n_r + M + n_t);
    IL_CHECK_CUDA(cudaFuncSetAttribute(k_ml, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    IL_REQUIRE(P < (1ll << 31), "too many problems");
    IL_LAUNCH(kProfOther, st,
              k_ml<<<(unsigned)P, kMlThreads, smem, st>>>(H, y, P, n_r, n_t, al, n_prefix, x_idx,
                                                          energy););
    IL_CHECK_CUDA(cudaGetLastError());
    return IL_OK;
}

}  // namespace il

namespace il {
int launch_ml_llr(const double* H, const double* y, const double* noise_var, int64_t P, int n_r,
                  int n_t, const Alphabet& al, double* llr, cudaStream_t st) {
    if (P == 0) return IL_OK;
    IL_REQUIRE(n_r <= kLlrMaxNr, "ML LLRs support n_r <= %d", kLlrMaxNr);
    const int M = al.m * al.m;
    int bpd = 0;
    while ((1 << bpd) < al.m) ++bpd;
    IL_REQUIRE(2 * bpd * n_t <= kLlrMaxBits && 2 * bpd <= kLlrMaxLast,
               "ML search space of %d bits exceeds the 24-bit guard", 2 * bpd * n_t);
    int64_t n_prefix = 1;
    for (int j = 0; j < n_t - 1; ++j) n_prefix *= M;
    const size_t smem = sizeof(cplx) * ((size_t)n_r * n_t + n_r + M);
    IL_CHECK_CUDA(cudaFuncSetAttribute(k_ml_llr, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    IL_REQUIRE(P < (1ll << 31), "too many problems");
    IL_LAUNCH(kProfOther, st,
              k_ml_llr<<<(unsigned)P, kMlThreads, smem, st>>>(H, y, noise_var, P, n_r, n_t, al,
                                                              n_prefix, bpd, llr););
    IL_CHECK_CUDA(cudaGetLastError());
    return IL_OK;
}
}  // namespace il
