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
