// Shared definitions for the isinglink-b200 CUDA library (sm_100a).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/isinglink_b200.h"

#define IL_HD __host__ __device__ __forceinline__
#define IL_D __device__ __forceinline__

namespace il {

// ---- error plumbing (C ABI: status codes + il_last_error) -----------------
void set_error(const char* fmt, ...);
int fail_cuda(cudaError_t e, const char* what);

#define IL_CHECK_CUDA(expr)                                   \
    do {                                                      \
        cudaError_t _e = (expr);                              \
        if (_e != cudaSuccess) return ::il::fail_cuda(_e, #expr); \
    } while (0)

#define IL_REQUIRE(cond, ...)                \
    do {                                     \
        if (!(cond)) {                       \
            ::il::set_error(__VA_ARGS__);    \
            return IL_ERR_ARG;               \
        }                                    \
    } while (0)

// ---- small complex FP64 helpers --------------------------------------------
struct cplx {
    double re, im;
};
IL_HD cplx cmul(cplx a, cplx b) { return {a.re * b.re - a.im * b.im, a.re * b.im + a.im * b.re}; }
// conj(a) * b
IL_HD cplx cmulc(cplx a, cplx b) { return {a.re * b.re + a.im * b.im, a.re * b.im - a.im * b.re}; }
IL_HD cplx cadd(cplx a, cplx b) { return {a.re + b.re, a.im + b.im}; }
IL_HD cplx csub(cplx a, cplx b) { return {a.re - b.re, a.im - b.im}; }
IL_HD double cabs2(cplx a) { return a.re * a.re + a.im * a.im; }

// Residual row r_k = y_k - sum_j H[k][j] x_j with every operation rounded
// explicitly (no contraction choices left to the compiler), so that every
// kernel computing ||y - Hx||^2 (linear.py:44-47) agrees bit-for-bit: the
// guess energy and the decoded-vector energy must tie exactly when the
// decision is unchanged (strict test, detector.py:52).
IL_D cplx resid_row(const cplx* Hk, const cplx* x, int n, cplx yk) {
    double sr = 0.0, si = 0.0;
    for (int j = 0; j < n; ++j) {
        const cplx a = Hk[j], b = x[j];
        sr = __dadd_rn(sr, __fma_rn(a.re, b.re, -__dmul_rn(a.im, b.im)));
        si = __dadd_rn(si, __fma_rn(a.re, b.im, __dmul_rn(a.im, b.re)));
    }
    return {__dsub_rn(yk.re, sr), __dsub_rn(yk.im, si)};
}
IL_D double abs2_rn(cplx a) { return __fma_rn(a.re, a.re, __dmul_rn(a.im, a.im)); }

// ---- warp helpers ----------------------------------------------------------
IL_D double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = __dadd_rn(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

// Constellation geometry passed to kernels by value.
struct Alphabet {
    int m;                 // PAM levels per dimension
    double spacing;        // level spacing (2c)
    double levels[32];     // ascending PAM levels
    double mids[31];       // (levels[k] + levels[k+1]) / 2, as channel.py:141-145
};

// Host: fill an Alphabet for square QAM (channel.py:88-108) or the VPP
// integer lattice 4*{-reach..reach} (precoder.py:79-90).
int make_qam_alphabet(int order, Alphabet* out);
int make_lattice_alphabet(int reach, Alphabet* out);

// Nearest-level index: number of midpoints strictly below v (searchsorted
// side="left"), so exact midpoints go to the smaller level.
IL_HD int level_index(double v, const Alphabet& al) {
    int k = 0;
    for (int i = 0; i < al.m - 1; ++i) k += (al.mids[i] < v) ? 1 : 0;
    return k;
}

}  // namespace il
