// Device helpers shared by the FP32 anneal kernels (anneal_fast.cu: legacy
// mma.sync coupling product; anneal_umma.cu: tcgen05 coupling product).
#pragma once
#include <cuda_fp16.h>

#include "il_internal.cuh"
#include "rng_numpy.cuh"

#ifndef IL_FHFMA_SPLIT  // f16 hi/lo split residual via mixed-precision FMA
#define IL_FHFMA_SPLIT 1
#endif
#ifndef IL_BOUND_FLOOR  // per-thread lower bound on e replaces per-spin floor checks
#define IL_BOUND_FLOOR 1
#endif

namespace il {
namespace fastk {

#ifndef IL_SCALED_X  // state stored as sqrt(dt) x: the Euler factor is one FMA
#define IL_SCALED_X 1
#endif

struct FastScalars {
    float alpha;    // 1 + dt (p - 1)
    float ndt;      // -dt
    float beta;     // 1 + dt zeta a
    float ndtz;     // -dt zeta
    float e_floor;
    float thr2;     // diverge_threshold^2
    double dt;
    double x0_lo, x0_range;
    U128 jump_mult[4], jump_add[4];  // [3]: PCG64 advance by half a stream ([0..2] unused)
    int f_mvm, n_steps;
    double sdt;   // sqrt(dt): scale of the stored state (IL_SCALED_X)
    float qthr;   // alpha - dt thr^2: q below it means |x| > thr (IL_SCALED_X)
    int b_valid;  // anneal rows per problem that enter the selection (screened energies)
    int b_out;    // anneal rows per problem whose steps / mvms are counted (PAD + counts)
    int full_steps;  // refreshes at steps < full_steps take the lo(v) x hi(G) pass too
    int64_t n_probs; // problems in the launch (PACK: the last warp may hold one)
    const double* gstats;  // [P][2] max |G|, sum |G| + sum |b| from the front end, or null
    int rng;               // il_rng
    float x0_lo_f, x0_range_f;  // IL_RNG_PHILOX: FP32 x0 = fmaf(range, u, lo)
};

__device__ __forceinline__ uint32_t h2_bits(__half2 h) { return *reinterpret_cast<uint32_t*>(&h); }

// hi + lo split of a float pair into two packed f16x2 words (x in the low half)
__device__ __forceinline__ void split_h2(float2 v, uint32_t& hi, uint32_t& lo) {
    const __half2 h = __float22half2_rn(v);
    hi = h2_bits(h);
#if IL_FHFMA_SPLIT
    // residual v - f32(hi) by a mixed-precision FMA straight from the f16
    // halves (hi * -1 + v, exact): 2 FHFMA instead of 2 HADD2.F32 + 1 FADD2
    float r0, r1;
    asm("{\n .reg .b16 a, b;\n mov.b32 {a, b}, %2;\n"
        " fma.rn.f32.f16 %0, a, %4, %3;\n"
        " fma.rn.f32.f16 %1, b, %4, %5;\n}"
        : "=f"(r0), "=f"(r1)
        : "r"(hi), "f"(v.x), "h"((unsigned short)0xBC00), "f"(v.y));
    lo = h2_bits(__float22half2_rn(make_float2(r0, r1)));
#else
    const float2 hf = __half22float2(h);
    const float2 r = __fadd2_rn(v, make_float2(-hf.x, -hf.y));
    lo = h2_bits(__float22half2_rn(r));
#endif
}

__device__ __forceinline__ void mma_f16(float (&d)[4], const uint32_t (&a)[4], uint32_t b0,
                                        uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
        "{%8,%9}, {%0,%1,%2,%3};"
        : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

__device__ __forceinline__ float max_nan3(float a, float b, float c) {
    float r;
    asm("max.NaN.f32 %0, %1, %2;" : "=f"(r) : "f"(a), "f"(b));
    asm("max.NaN.f32 %0, %0, %1;" : "+f"(r) : "f"(c));
    return r;
}
__device__ __forceinline__ float max_nan(float a, float b) {
    float r;
    asm("max.NaN.f32 %0, %1, %2;" : "=f"(r) : "f"(a), "f"(b));
    return r;
}

// One explicit-Euler step of a spin pair (packed FP32x2).
//   x' = x (alpha - dt x^2) + e C      (C = -dt eps c)
//   e' = max(e_floor, e (beta - dt zeta x^2))
// x2 of the incoming state is folded into the divergence max.
template <bool SAME_QR>
__device__ __forceinline__ void euler_pair(float2& x, float2& e, const float2 C,
                                           const FastScalars& s, float e_floor, float& dv) {
    const float2 x2 = __fmul2_rn(x, x);
    dv = max_nan3(dv, x2.x, x2.y);
    const float2 q = __ffma2_rn(make_float2(s.ndt, s.ndt), x2, make_float2(s.alpha, s.alpha));
    // at the default operating point (zeta = 1, p - 1 = a) the x and e
    // factors coincide exactly and one packed FMA is saved
    const float2 r = SAME_QR ? q
                             : __ffma2_rn(make_float2(s.ndtz, s.ndtz), x2, make_float2(s.beta, s.beta));
    const float2 t = __fmul2_rn(x, q);
    x = __ffma2_rn(e, C, t);
    const float2 er = __fmul2_rn(e, r);
#if IL_BOUND_FLOOR
    // floor applied by the caller only if some e of the step may fall below it
    e = er;
    (void)e_floor;
#else
    e = make_float2(fmaxf(er.x, e_floor), fmaxf(er.y, e_floor));
#endif
}

__device__ __forceinline__ float2 floor2(float2 e, float f) {
    return make_float2(fmaxf(e.x, f), fmaxf(e.y, f));
}

template <bool SAME_QR>
__device__ __forceinline__ void euler_one(float& x, float& e, const float C, const FastScalars& s,
                                          float e_floor, float& dv) {
    const float x2 = x * x;
    dv = max_nan(dv, x2);
    const float q = fmaf(s.ndt, x2, s.alpha);
    const float r = SAME_QR ? q : fmaf(s.ndtz, x2, s.beta);
    x = fmaf(e, C, x * q);
    e = fmaxf(e * r, e_floor);
}

__device__ __forceinline__ float min_nan3(float a, float b, float c) {
    float r;
    asm("min.NaN.f32 %0, %1, %2;" : "=f"(r) : "f"(a), "f"(b));
    asm("min.NaN.f32 %0, %0, %1;" : "+f"(r) : "f"(c));
    return r;
}
__device__ __forceinline__ float min_nan(float a, float b) {
    float r;
    asm("min.NaN.f32 %0, %1, %2;" : "=f"(r) : "f"(a), "f"(b));
    return r;
}

// Scaled-state Euler step (IL_SCALED_X, x- and e-factors equal): with
// x~ = sqrt(dt) x the factor q = 1 + dt (p - 1) - dt x^2 = alpha - x~^2 is a
// single FMA (x^2 is never formed), and |x| > thr <=> q < alpha - dt thr^2,
// so the divergence test tracks the sticky NaN-propagating minimum of q.
// The coupling term scales with the state (C~ = sqrt(dt) C is what the
// refresh produces from x~), so x~' = x~ q + e C~.
__device__ __forceinline__ void euler_pair_sc(float2& x, float2& e, const float2 C, float alpha,
                                              float& qmin) {
    const float2 q = __ffma2_rn(make_float2(-x.x, -x.y), x, make_float2(alpha, alpha));
    qmin = min_nan3(qmin, q.x, q.y);
    x = __ffma2_rn(e, C, __fmul2_rn(x, q));
    e = __fmul2_rn(e, q);
}
__device__ __forceinline__ void euler_one_sc(float& x, float& e, const float C, float alpha,
                                             float e_floor, float& qmin) {
    const float q = fmaf(-x, x, alpha);
    qmin = min_nan(qmin, q);
    x = fmaf(e, C, x * q);
    e = fmaxf(e * q, e_floor);
}

// PCG64 advance-by-k constants: state_k = M^k state_0 + inc * (M^{k-1} + ... + 1)
inline void pcg_jump(int k, U128* mult, U128* add) {
    const U128 M = {0x2360ED051FC65DA4ull, 0x4385DF649FCCF645ull};
    U128 pm = {0, 1}, sum = {0, 0};
    for (int i = 0; i < k; ++i) {
        sum = add128(sum, pm);
        pm = mul128(pm, M);
    }
    *mult = pm;
    *add = sum;
}


}  // namespace fastk
}  // namespace il
