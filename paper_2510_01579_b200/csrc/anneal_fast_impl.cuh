// Template of the throughput anneal kernel (k_anneal_fast) and its launch
// chain; anneal_fast_nt<k>.cu instantiate it per register layout NT (so that
// the layouts compile in parallel) and anneal_fast.cu dispatches.
#pragma once
// Throughput CIM-CAC anneal kernel: FP32 state in registers, coupling
// product on the tensor cores, state never leaves the register file.
//
// Dynamics (reference _kernel.pyx:64-97):
//   every f_mvm steps:  m = G (x1 + x2);  c1 = m - g.x1 + b xa;  c2 = m - g.x2 + b xa;
//                       c_aux = b.(x1 + x2)
//   every step:         x += dt((p-1)x - x^3 - eps e c);   e = max(e_floor, e - dt zeta (x^2 - a) e)
//
// Mapping (one warp = 16 anneals of one problem, N = 8*NT spins per half):
//   The refresh is the small GEMM  M^T[a][i] = sum_j V^T[a][j] G[j][i]  with
//   a = anneal (MMA M dimension), i = spin (N dimension), j = spin (K), issued
//   as mma.sync.m16n8k16 f16 tiles with FP32 accumulate.  Thread (g = lane/4,
//   t = lane%4) owns anneals {g, g+8} and, in every n-tile n, spins {8n+2t,
//   8n+2t+1} of both halves: exactly the accumulator (C) fragment of the tile.
//   The A fragment of k-tile k holds the thread's columns {2t, 2t+1, 2t+8,
//   2t+9}, i.e. spins {16k+2t, +1} and {16k+8+2t, +1}: n-tiles 2k and 2k+1 of
//   the thread's own spins.  G's B fragments are staged once per problem, so
//   a refresh moves no data between lanes: v = x1 + x2 is formed in
//   registers, fed to the MMA, and the result lands where the Euler update
//   needs it.
//   IL_PREC_FP32 splits both operands into f16 hi + lo parts (3 MMAs per
//   tile: hi*hi + lo*hi + hi*lo) for FP32-level accuracy; IL_PREC_TF32 uses
//   one pass.  The Euler update runs on packed FP32x2 (FFMA2/FMUL2) over spin
//   pairs; at the reference operating point the state is stored as sqrt(dt) x
//   (IL_SCALED_X) so that the update is 4 packed ops per pair.  The aux spin
//   (one per anneal) is integrated redundantly and bit-identically by the 4
//   lanes of a quad; c_aux comes from a quad shuffle reduction.
//
// Divergence: a per-anneal sticky NaN-propagating extremum (max of x^2, or
// the min of the scaled factor q), matching the reference's `diverged` flag;
// spins of a diverged anneal are not frozen at the halting step, which is
// harmless because diverged anneals are excluded from selection
// (solver.py:262-264).  The exact kernel serves the drop-in run_anneals path
// where frozen spins are part of the contract.
//
// Energies: every anneal's in FP64, or (the detection path) an FP32
// tensor-core screen with FP64 for the anneals that can be the argmin.
//
// Scaling: G, g, b are pre-multiplied by -dt*eps so that the MMA directly
// yields the -dt*eps*c term of the update.
#include <cuda_fp16.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <type_traits>

#include "il_internal.cuh"
#include "rng_numpy.cuh"
#include "rng_philox.cuh"
#include "il_anneal.cuh"

namespace il {
namespace fast_impl {
using namespace fastk;

#ifndef IL_FAST_WARPS  // warps per CTA (2 warps = one problem at 32 anneals)
#define IL_FAST_WARPS 4
#endif
constexpr int kWarpsPerCta = IL_FAST_WARPS;
#ifndef IL_FAST_MINB  // CTAs per SM (4-warp CTAs) for 16 < N <= 32
#define IL_FAST_MINB 3
#endif
#ifndef IL_FAST_MINB2  // CTAs per SM for N <= 16
#define IL_FAST_MINB2 4
#endif
#ifndef IL_STEP_UNROLL  // unroll factor of the step loop
#define IL_STEP_UNROLL 2
#endif
constexpr int kStepUnroll = IL_STEP_UNROLL;
constexpr int kRefCount = 0, kRefYes = 1, kRefNo = 2;  // refresh modes of a step
#ifndef IL_PAIRS_NT_MASK  // register layouts NT (bit NT) whose f_mvm = 2 loop runs as step pairs
#define IL_PAIRS_NT_MASK 0x1FE  // every layout NT = 1-8 (tools/gpu/ab_large_nt.sh)
#endif
#ifndef IL_PAIR_UNROLL2_MAX_NT  // layouts NT <= this run two step pairs per loop iteration
#define IL_PAIR_UNROLL2_MAX_NT 2  // 8x8 anneal 1.904 -> 1.882 ms; NT = 3, 4 spill at 2
#endif



template <int NT, bool PACK>
struct FastLayout {
    static constexpr int N = 8 * NT;
    static constexpr int S = 2 * N + 1;
    static constexpr int KT = (NT + 1) / 2;               // k16 tiles of the f16 MMA
    static constexpr int NP = PACK ? 2 : 1;               // problems per warp
    static constexpr int kFragF4 = KT * NT * 32;          // uint4 per problem
    static constexpr int kX0F4 = (16 * S + 3) / 4;        // x0 staging, aliased
    // + one uint4 of per-warp scalars kept out of registers during the loop
    // + NP x NT x 32 uint4 of per-lane refresh constants {Kg, -Kb}
    static constexpr int kKgF4 = (NP * kFragF4 > kX0F4 ? NP * kFragF4 : kX0F4) + 1;
    static constexpr int kWarpF4 = kKgF4 + NP * NT * 32;
    static constexpr size_t kWarpBytes = sizeof(float4) * kWarpsPerCta * kWarpF4;
};

// Tensor-core operand scaling.  The coupling product runs on f16 operands
// (11-bit significand, like TF32, at twice the K per instruction).  To keep
// the lo parts of the split out of the f16 subnormal range, -K*G is scaled
// by 2^sc per problem so that its largest entry lies in [128, 256).  The
// scale is carried, exactly, by the error variables: every coupling term
// enters the update as e*C, so storing e_s = e * 2^-sc and C_s = C * 2^sc
// leaves e*C unchanged, and e' = max(floor, e r) becomes
// e_s' = max(floor * 2^-sc, e_s r) -- power-of-two scalings are exact.
//
// PAD: the problems have n_rt < N spins per half (any n_rt, e.g. odd n_t or
// n_t = 20, 28).  The register layout stays that of N; spins n_rt..N-1 of
// each half are inert: zero rows and columns of G, zero g and b, and an
// initial state of exactly 0, which the dynamics keep at 0 (x' = x q + e C
// with x = C = 0), so they neither couple nor diverge.  Global memory is
// addressed with n_rt (G [n_rt][n_rt], spins [2 n_rt + 1]), and the initial
// states are the same stream draws as for an unpadded problem of n_rt spins.
// The PAD instantiations also serve the instrumented calls: with steps_out
// non-null they count, per anneal, the steps before the first divergence
// (the reference's `steps`, _kernel.pyx:85-97) and the coupling refreshes
// (`mvms`), for the first s.b_out rows of each problem ([P][b_out] layout).
//
// PACK: problems of 8 anneals (n_anneals <= 8).  A warp carries two of them,
// 2 task and 2 task + 1: accumulator rows g are the first problem's anneals,
// rows g + 8 the second's.  Every per-problem quantity (scale, fragments,
// refresh constants, floors, energies) is indexed by the row half h; the
// coupling product runs once per problem (two MMA sets over the same A
// fragments, each keeping its own half of the rows), so the Euler work is
// not spent on padding rows.
template <int NT, bool SPLIT, bool SAME_QR, bool PAD, bool PACK>
__global__ void __launch_bounds__(kWarpsPerCta * 32,
                                  (NT <= 2 ? IL_FAST_MINB2 : (NT <= 4 ? IL_FAST_MINB : 1)) * 4 / kWarpsPerCta)
k_anneal_fast(const double* __restrict__ Gall, const double* __restrict__ gall,
              const double* __restrict__ ball, const uint64_t* __restrict__ base_seed,
              const double* __restrict__ eps_p, int64_t n_tasks, int tiles_per_prob,
              FastScalars s, int8_t* __restrict__ spins, uint8_t* __restrict__ diverged,
              double* __restrict__ energies, bool screened, int n_rt,
              int64_t* __restrict__ steps_out, int64_t* __restrict__ mvms_out) {
    using L = FastLayout<NT, PACK>;
    constexpr int N = L::N;
    constexpr int S = L::S;
    constexpr int KT = L::KT;
    constexpr int NP = L::NP;
    const int nr = PAD ? n_rt : N;  // spins per half in global memory
    const int Sg = 2 * nr + 1;       // spins per anneal in global memory
    // scaled state (IL_SCALED_X): x~ = sqrt(dt) x wherever x is stored
    constexpr bool SC = IL_SCALED_X && SAME_QR;
    extern __shared__ __align__(16) uint4 smem_u4[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t task = (int64_t)blockIdx.x * kWarpsPerCta + warp;
    const bool valid = task < n_tasks;
    const int64_t prob = PACK ? 2 * task : task / tiles_per_prob;
    const int mt = PACK ? 0 : (int)(task % tiles_per_prob);
    const int B = PACK ? 8 : tiles_per_prob * 16;
    const int g = lane >> 2, t = lane & 3;
    const int hown = t & 1;  // the aux spin of anneal g + 8*hown is integrated by this lane
    // problem of row half h (PACK), whether its outputs are written (a
    // missing second problem of the last warp computes a copy of the first)
    int64_t probh[2] = {prob, prob};
    bool hval[2] = {true, true};
    if constexpr (PACK) {
        hval[1] = prob + 1 < s.n_probs;
        probh[1] = hval[1] ? prob + 1 : prob;
    }
    const int64_t rowh[2] = {PACK ? probh[0] * 8 + g : prob * (int64_t)B + mt * 16 + g,
                             PACK ? probh[1] * 8 + g : prob * (int64_t)B + mt * 16 + g + 8};

    const double* Gq[NP];
    const double* gq[NP];
    const double* bq[NP];
#pragma unroll
    for (int q = 0; q < NP; ++q) {
        Gq[q] = Gall + probh[q] * (int64_t)nr * nr;
        gq[q] = gall + probh[q] * nr;
        bq[q] = ball + probh[q] * nr;
    }
    const double* G = Gq[0];
    const double* gv_p = gq[0];
    const double* bv_p = bq[0];
    if (!valid) return;
    // G, g and b are first read by the fragment staging after the x0 replay:
    // start pulling their lines into L2 now, behind the replay's arithmetic
    // (4.10 -> 4.07 ms per 16x16 slot)
#pragma unroll
    for (int q = 0; q < NP; ++q) {
        for (int i = 16 * lane; i < nr * nr; i += 512)
            asm volatile("prefetch.global.L2 [%0];" ::"l"(Gq[q] + i));
        if (lane < 2) {
            asm volatile("prefetch.global.L2 [%0];" ::"l"(lane ? bq[q] : gq[q]));
            if (nr > 16) asm volatile("prefetch.global.L2 [%0];" ::"l"((lane ? bq[q] : gq[q]) + 16));
        }
    }
    uint4* frag = smem_u4 + warp * L::kWarpF4;      // G fragments (after x0 is consumed)
    float* x0s = reinterpret_cast<float*>(frag);    // x0 staging [16][S]

    // ---- initial states: replayed NumPy streams (or Philox), 2 lanes per anneal
    {
        const int al = lane & 15, part = lane >> 4;
        const int a = PACK ? (al & 7) : mt * 16 + al;
        if (s.rng == IL_RNG_PHILOX) {
            // counter-based: lane part p draws the 4-blocks p, p + 2, ...
            float* row = x0s + al * S;
            if constexpr (PAD)
                for (int i = nr + part; i < N; i += 2) row[i] = row[N + i] = 0.f;
            const uint64_t sd = base_seed[PACK ? probh[al >> 3] : prob];
            for (int blk = part; 4 * blk < Sg; blk += 2) {
                float v[4];
                philox_x0_block(sd, (uint32_t)a, (uint32_t)blk, s.x0_lo_f, s.x0_range_f, v);
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const int i = 4 * blk + q;
                    if (i < Sg) {
                        const int pos = !PAD ? i : (i < nr ? i : (i < 2 * nr ? N + i - nr : 2 * N));
                        row[pos] = SC ? (float)(s.sdt * (double)v[q]) : v[q];
                    }
                }
            }
        } else {
            Pcg64 rng;
            rng.seed_from(derive_seed2(base_seed[PACK ? probh[al >> 3] : prob], (uint64_t)a));
            // lane part 1 jumps ahead over the first half of the stream
            if (part) rng.state = add128(mul128(rng.state, s.jump_mult[3]), mul128(rng.inc, s.jump_add[3]));
            if constexpr (PAD) {
                // stream draw i -> padded position (half A, half B, aux); the
                // inert positions start at exactly 0
                float* row = x0s + al * S;
                for (int i = nr + part; i < N; i += 2) row[i] = row[N + i] = 0.f;
                const int S0 = (Sg + 1) / 2;
                const int i0 = part ? S0 : 0, i1 = part ? Sg : S0;
                for (int i = i0; i < i1; ++i) {
                    const double u = rng.uniform(s.x0_lo, s.x0_range);
                    row[i < nr ? i : (i < 2 * nr ? N + i - nr : 2 * N)] = SC ? (float)(s.sdt * u) : (float)u;
                }
            } else {
                constexpr int S0 = (S + 1) / 2;
                const int i0 = part ? S0 : 0, i1 = part ? S : S0;
                for (int i = i0; i < i1; ++i)
                    x0s[al * S + i] = SC ? (float)(s.sdt * rng.uniform(s.x0_lo, s.x0_range))
                                         : (float)rng.uniform(s.x0_lo, s.x0_range);
            }
        }
    }

    // ---- per-problem scale 2^sc for -K*G ------------------------------------
    double Ksq[NP];
    float e_initq[NP], e_floorq[NP];
#pragma unroll
    for (int q = 0; q < NP; ++q) {
        const double K = s.dt * eps_p[probh[q]];
        const double* Gp = Gq[q];
        double gmax = 0.0;
        if (s.gstats) {
            // precomputed by the front end (k_front_rows) while it held the rows
            gmax = s.gstats[2 * probh[q]];
            if (screened && lane == 0)
                reinterpret_cast<double*>(frag + L::kKgF4 - 1)[q] = s.gstats[2 * probh[q] + 1];
        } else if (screened) {
            double mag = 0.0;  // sum |G| + sum |b|: the screen bound, parked in shared memory
#pragma unroll 4
            for (int i = lane; i < nr * nr; i += 32) {
                const double v = fabs(__ldg(Gp + i));
                gmax = fmax(gmax, v);
                mag += v;
            }
            for (int i = lane; i < nr; i += 32) mag += fabs(bq[q][i]);
            mag = warp_sum(mag);
            if (lane == 0) reinterpret_cast<double*>(frag + L::kKgF4 - 1)[q] = mag;
        } else {
#pragma unroll 4
            for (int i = lane; i < nr * nr; i += 32) gmax = fmax(gmax, fabs(__ldg(Gp + i)));
        }
        if (!s.gstats) {
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) gmax = fmax(gmax, __shfl_xor_sync(0xffffffffu, gmax, o));
        }
        int ex = 0;
        frexp(K * gmax, &ex);
        const int sc = (K * gmax > 0.0) ? 8 - ex : 0;
        Ksq[q] = ldexp(K, sc);
        e_initq[q] = ldexpf(1.0f, -sc);
        e_floorq[q] = ldexpf(s.e_floor, -sc);
    }
    const double Ks = Ksq[0];
    const float e_init = e_initq[0];
    const float e_floor = e_floorq[0];

    __syncwarp();
    float2 xA[2][NT], xB[2][NT], eA[2][NT], eB[2][NT], CA[2][NT], CB[2][NT];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        const float* r = x0s + (g + 8 * h) * S;
#pragma unroll
        for (int n = 0; n < NT; ++n) {
            const int i = 8 * n + 2 * t;
            xA[h][n] = make_float2(r[i], r[i + 1]);
            xB[h][n] = make_float2(r[N + i], r[N + i + 1]);
            eA[h][n] = eB[h][n] = make_float2(e_initq[PACK ? h : 0], e_initq[PACK ? h : 0]);
            CA[h][n] = CB[h][n] = make_float2(0.f, 0.f);
        }
    }
    // divergence tracking: sticky max of x^2, or (SC) sticky min of q
    constexpr float kD0 = SC ? INFINITY : 0.f;
    float xa = x0s[(g + 8 * hown) * S + 2 * N], ea = e_initq[PACK ? hown : 0], Ca = 0.f, dva = kD0;
    float dv[2][2] = {{kD0, kD0}, {kD0, kD0}};
#if IL_BOUND_FLOOR
    float e_lb = e_init;  // lower bound of every eA/eB of this thread
    [[maybe_unused]] float e_lbh[2] = {e_initq[0], e_initq[NP - 1]};  // PACK: per row half
#endif
    __syncwarp();

    // ---- stage -Ks*G as f16 B fragments (hi, lo) of m16n8k16 --------------
    // b0 = B[16kt+2t, +1][8n+g], b1 = B[16kt+8+2t, +1][8n+g]; rows >= N are zero
#pragma unroll
    for (int pq = 0; pq < NP; ++pq) {
        const double* Gp = Gq[pq];
        const double Kp = Ksq[pq];
#pragma unroll
        for (int kt = 0; kt < KT; ++kt) {
#pragma unroll
            for (int n = 0; n < NT; ++n) {
                const int c = 8 * n + g;
                float f[4];
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const int r = 16 * kt + 2 * t + (q & 1) + 8 * (q >> 1);
                    f[q] = (r < nr && c < nr) ? (float)(-Kp * __ldg(Gp + r * nr + c)) : 0.f;
                }
                uint32_t h01, l01, h23, l23;
                split_h2(make_float2(f[0], f[1]), h01, l01);
                split_h2(make_float2(f[2], f[3]), h23, l23);
                frag[pq * L::kFragF4 + (kt * NT + n) * 32 + lane] = make_uint4(h01, h23, l01, l23);
            }
        }
    }
    // per-thread spin constants Ks g_i and -Ks b_i for spins 8n+2t+{0,1}: kept
    // in shared memory and re-read at every refresh (the registers go to the
    // Euler update's scheduling instead)
    float4* kgs = reinterpret_cast<float4*>(frag + L::kKgF4);
#pragma unroll
    for (int pq = 0; pq < NP; ++pq) {
        const double Kp = Ksq[pq];
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) {
            const int i = 8 * nt + 2 * t;
            const double g0 = i < nr ? gq[pq][i] : 0.0, g1 = i + 1 < nr ? gq[pq][i + 1] : 0.0;
            const double b0 = i < nr ? bq[pq][i] : 0.0, b1 = i + 1 < nr ? bq[pq][i + 1] : 0.0;
            kgs[(pq * NT + nt) * 32 + lane] = make_float4((float)(Kp * g0), (float)(Kp * g1),
                                                          (float)(-Kp * b0), (float)(-Kp * b1));
        }
    }
    // constants of row half h's problem
    auto kg4 = [&](int h, int n) {
        float4 r;
        asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
                     : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w)
                     : "r"(smem_u32(kgs + ((PACK ? h : 0) * NT + n) * 32 + lane)));
        return r;
    };
    auto nkb = [&](int h, int n) {
        const float4 r = kg4(h, n);
        return make_float2(r.z, r.w);
    };
    __syncwarp();

    // PAD + counts: iterations whose incoming states were all below the
    // threshold (sticky tracking, so the count stops at the first divergence)
    [[maybe_unused]] int cnt[2] = {0, 0};
    const bool counting = PAD && steps_out != nullptr;
    int until_refresh = 0;
    // One step; FULL_C selects the refresh precision (std::true_type: all
    // three split passes, std::false_type: the lo(v) x hi(G) pass dropped).
    // REF_C: kRefCount (refresh when the countdown reaches 0), kRefYes /
    // kRefNo (the caller knows the step's phase: f_mvm = 2 pair loops).
    auto step_body = [&](auto full_c, auto ref_c) {
        constexpr bool FULL = decltype(full_c)::value;
        constexpr int REF = decltype(ref_c)::value;
        if (REF == kRefYes || (REF == kRefCount && until_refresh == 0)) {
            if constexpr (REF == kRefCount) until_refresh = s.f_mvm;
            // ---- refresh: v = x1 + x2, M' = -Ks G v on tensor cores -----------
            float2 v[2][NT];
            float pb[2] = {0.f, 0.f};
            // packed partial sums of -Ks b.v over the thread's spin pairs; every
            // lane of a quad sums the same pairs in the same order, so the two
            // owner lanes of an aux spin still agree bit for bit
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                float2 p2 = make_float2(0.f, 0.f);
#pragma unroll
                for (int n = 0; n < NT; ++n) {
                    v[h][n] = __fadd2_rn(xA[h][n], xB[h][n]);
                    p2 = __ffma2_rn(nkb(h, n), v[h][n], p2);
                }
                pb[h] = p2.x + p2.y;
            }
            // aux states of both anneals of the quad, from their owner lanes
            const float xa0 = __shfl_sync(0xffffffffu, xa, (lane & ~3) | 0);
            const float xa1 = __shfl_sync(0xffffffffu, xa, (lane & ~3) | 1);
            {
                const float mine = hown ? pb[1] : pb[0];
                const float other = hown ? pb[0] : pb[1];
                // quad sum of the own anneal's partials; the two owner lanes of an
                // anneal (t, t^2) add the same four terms in commuted order, so
                // their aux trajectories stay bit-identical
                float tot = mine + __shfl_xor_sync(0xffffffffu, other, 1);
                tot += __shfl_xor_sync(0xffffffffu, tot, 2);
                Ca = tot;
            }
            float acc[NT][4];
#pragma unroll
            for (int n = 0; n < NT; ++n) acc[n][0] = acc[n][1] = acc[n][2] = acc[n][3] = 0.f;
            // A fragment of k-tile kt: a0 = (g, 2t..), a1 = (g+8, 2t..), a2 = (g, 2t+8..), a3 = (g+8, 2t+8..)
            auto a_frag = [&](int kt, uint32_t (&ahi)[4], uint32_t (&alo)[4]) {
                if (SPLIT && FULL) {
                    split_h2(v[0][2 * kt], ahi[0], alo[0]);
                    split_h2(v[1][2 * kt], ahi[1], alo[1]);
                    if (2 * kt + 1 < NT) {
                        split_h2(v[0][2 * kt + 1], ahi[2], alo[2]);
                        split_h2(v[1][2 * kt + 1], ahi[3], alo[3]);
                    } else {
                        ahi[2] = ahi[3] = alo[2] = alo[3] = 0u;
                    }
                } else {
                    ahi[0] = h2_bits(__float22half2_rn(v[0][2 * kt]));
                    ahi[1] = h2_bits(__float22half2_rn(v[1][2 * kt]));
                    ahi[2] = 2 * kt + 1 < NT ? h2_bits(__float22half2_rn(v[0][2 * kt + 1])) : 0u;
                    ahi[3] = 2 * kt + 1 < NT ? h2_bits(__float22half2_rn(v[1][2 * kt + 1])) : 0u;
                }
            };
            auto mma_tile = [&](float (&d)[4], const uint32_t (&ahi)[4], const uint32_t (&alo)[4],
                                const uint4 f) {
                if (SPLIT) {
                    if (FULL) mma_f16(d, alo, f.x, f.y);
                    mma_f16(d, ahi, f.z, f.w);
                }
                mma_f16(d, ahi, f.x, f.y);
            };
            if constexpr (!PACK) {
#pragma unroll
                for (int kt = 0; kt < KT; ++kt) {
                    uint32_t ahi[4], alo[4];
                    a_frag(kt, ahi, alo);
#pragma unroll
                    for (int n = 0; n < NT; ++n) mma_tile(acc[n], ahi, alo, frag[(kt * NT + n) * 32 + lane]);
                }
            } else {
                // one product per problem over the same A fragments; rows g
                // keep the first problem's result, rows g + 8 the second's
                uint32_t ahi[KT][4], alo[KT][4];
#pragma unroll
                for (int kt = 0; kt < KT; ++kt) a_frag(kt, ahi[kt], alo[kt]);
                float keep[NT][2];
#pragma unroll
                for (int pq = 0; pq < 2; ++pq) {
                    if (pq) {
#pragma unroll
                        for (int n = 0; n < NT; ++n) {
                            keep[n][0] = acc[n][0];
                            keep[n][1] = acc[n][1];
                            acc[n][0] = acc[n][1] = acc[n][2] = acc[n][3] = 0.f;
                        }
                    }
#pragma unroll
                    for (int kt = 0; kt < KT; ++kt)
#pragma unroll
                        for (int n = 0; n < NT; ++n)
                            mma_tile(acc[n], ahi[kt], alo[kt],
                                     frag[pq * L::kFragF4 + (kt * NT + n) * 32 + lane]);
                }
#pragma unroll
                for (int n = 0; n < NT; ++n) {
                    acc[n][0] = keep[n][0];
                    acc[n][1] = keep[n][1];
                }
            }
            // ---- coupling assembly: C_s = M' + Ks g x_self - Ks b xa ----------
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const float xah = h ? xa1 : xa0;
#pragma unroll
                for (int n = 0; n < NT; ++n) {
                    const float2 m2 = make_float2(acc[n][2 * h], acc[n][2 * h + 1]);
                    const float4 kk = kg4(h, n);
                    const float2 u2 = __ffma2_rn(make_float2(kk.z, kk.w), make_float2(xah, xah), m2);
                    CA[h][n] = __ffma2_rn(make_float2(kk.x, kk.y), xA[h][n], u2);
                    CB[h][n] = __ffma2_rn(make_float2(kk.x, kk.y), xB[h][n], u2);
                }
            }
        }
#pragma unroll
        for (int h = 0; h < 2; ++h) {
#pragma unroll
            for (int n = 0; n < NT; ++n) {
                if constexpr (SC) {
                    euler_pair_sc(xA[h][n], eA[h][n], CA[h][n], s.alpha, dv[h][n & 1]);
                    euler_pair_sc(xB[h][n], eB[h][n], CB[h][n], s.alpha, dv[h][n & 1]);
                } else {
                    const float ef = e_floorq[PACK ? h : 0];
                    euler_pair<SAME_QR>(xA[h][n], eA[h][n], CA[h][n], s, ef, dv[h][n & 1]);
                    euler_pair<SAME_QR>(xB[h][n], eB[h][n], CB[h][n], s, ef, dv[h][n & 1]);
                }
            }
        }
#if IL_BOUND_FLOOR
        // e' = max(e_floor, e r).  Every e of this thread stays >= e_lb, a
        // lower bound advanced per step with the smallest factor any of its
        // spins can have: r_i = fma(-dt zeta, x2_i, beta) >= fma(-dt zeta, dmax,
        // beta) since x2_i <= dmax (the sticky max of x^2 already tracked for
        // divergence) and rounding is monotone.  While e_lb r_lb >= e_floor no
        // floor can bind and the 2 FMNMX per spin pair are skipped; otherwise
        // every element is clamped exactly as before (also for NaN).  The branch
        // is warp-uniform (a vote): in a clamp round the lanes whose bound
        // holds clamp too, a no-op for them (e >= nxt >= e_floor, no NaN:
        // a NaN factor makes the bound NaN), so no convergence barrier is
        // needed (4.055 -> 4.043 ms per 16x16 slot).
        if constexpr (PACK) {
            // one bound per row half (the halves have their own floors)
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const float r_lb = SC ? min_nan(dv[h][0], dv[h][1])
                                      : (SAME_QR ? fmaf(s.ndt, max_nan(dv[h][0], dv[h][1]), s.alpha)
                                                 : fmaf(s.ndtz, max_nan(dv[h][0], dv[h][1]), s.beta));
                const float nxt = e_lbh[h] * r_lb;
                const bool fine = nxt >= e_floorq[h];
                if (__all_sync(0xffffffffu, fine)) {
                    e_lbh[h] = nxt;
                } else {
#pragma unroll
                    for (int n = 0; n < NT; ++n) {
                        eA[h][n] = floor2(eA[h][n], e_floorq[h]);
                        eB[h][n] = floor2(eB[h][n], e_floorq[h]);
                    }
                    e_lbh[h] = fine ? nxt : e_floorq[h];
                }
            }
        } else {
            // (SC: the sticky minimum of q is itself the smallest factor)
            const float r_lb = SC ? min_nan3(min_nan(dv[0][0], dv[0][1]), dv[1][0], dv[1][1])
                                  : [&] {
                                        const float dmax = max_nan3(max_nan(dv[0][0], dv[0][1]),
                                                                    dv[1][0], dv[1][1]);
                                        return SAME_QR ? fmaf(s.ndt, dmax, s.alpha)
                                                       : fmaf(s.ndtz, dmax, s.beta);
                                    }();
            const float nxt = e_lb * r_lb;
            // warp-uniform branch (no convergence barrier): in the rare clamp
            // round every lane clamps -- a no-op where e >= nxt >= e_floor
            const bool fine = nxt >= e_floor;
            if (__all_sync(0xffffffffu, fine)) {
                e_lb = nxt;
            } else {
#pragma unroll
                for (int h = 0; h < 2; ++h)
#pragma unroll
                    for (int n = 0; n < NT; ++n) {
                        eA[h][n] = floor2(eA[h][n], e_floor);
                        eB[h][n] = floor2(eB[h][n], e_floor);
                    }
                e_lb = fine ? nxt : e_floor;
            }
        }
#endif
        if constexpr (SC)
            euler_one_sc(xa, ea, Ca, s.alpha, e_floorq[PACK ? hown : 0], dva);
        else
            euler_one<SAME_QR>(xa, ea, Ca, s, e_floorq[PACK ? hown : 0], dva);
        if constexpr (PAD) {
            if (counting) {
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    float d = SC ? min_nan(dv[h][0], dv[h][1]) : max_nan(dv[h][0], dv[h][1]);
                    if (h == hown) d = SC ? min_nan(d, dva) : max_nan(d, dva);
                    cnt[h] += SC ? (d >= s.qthr) : (d <= s.thr2);
                }
            }
        }
        if constexpr (REF == kRefCount) --until_refresh;
    };
    // the refreshes of steps < s.full_steps carry all three passes, the later
    // ones two (two loops, so that neither carries a branch on the mode)
    using RefYes = std::integral_constant<int, kRefYes>;
    using RefNo = std::integral_constant<int, kRefNo>;
    using RefCount = std::integral_constant<int, kRefCount>;
    const int n_full = min(s.full_steps, s.n_steps);
    // f_mvm = 2 (the reference's default): steps [a, b), a even, as pairs
    // (refresh + step, step) whose refresh is known at compile time -- no
    // countdown and no refresh branch: 16x16 slot anneal 4.010 -> 3.976 ms,
    // 8x8 1.953 -> 1.909, N_a = 8 1.444 -> 1.385, n_t = 12 3.186 -> 3.030,
    // n_t = 20 / 24 / 28 / 32 6.24 / 7.34 / 9.82 / 12.79 -> 6.02 / 7.20 /
    // 9.32 / 10.87, bit-identical.  Two pairs per iteration only for NT <= 2
    // (8x8 anneal 1.904 -> 1.882 ms); for NT >= 3 they spill.
    constexpr int kPairUnroll = NT <= IL_PAIR_UNROLL2_MAX_NT ? 2 : 1;
    auto pairs = [&](auto full_c, int a, int b) {
        int step = a;
#pragma unroll kPairUnroll
        for (; step + 1 < b; step += 2) {
            step_body(full_c, RefYes{});
            step_body(full_c, RefNo{});
        }
        if (step < b) step_body(full_c, RefYes{});
    };
    // any other f_mvm: the countdown (the all-three-pass loop unrolled by 4
    // for the one-problem layouts NT = 3, 4: 0.5% faster there; at NT >= 5
    // the unrolled countdown also slowed the pairs loop beside it: n_t = 20
    // anneal 6.60 vs 6.02 ms)
    constexpr int kUnrollFull = (PACK || NT <= 2 || NT >= 5) ? kStepUnroll : 2 * kStepUnroll;
    constexpr bool kPairs = (IL_PAIRS_NT_MASK >> NT) & 1;
    if (kPairs && s.f_mvm == 2 && (n_full & 1) == 0) {
        pairs(std::true_type{}, 0, n_full);
        pairs(std::false_type{}, n_full, s.n_steps);
    } else {
#pragma unroll kUnrollFull
        for (int step = 0; step < n_full; ++step) step_body(std::true_type{}, RefCount{});
#pragma unroll kStepUnroll
        for (int step = n_full; step < s.n_steps; ++step) step_body(std::false_type{}, RefCount{});
    }

    // ---- epilogue: divergence flags, spins, FP64 energies --------------------
    // E = u'Gu - 2 tr G + 2 s_aux b'u with u = s_A + s_B (solver.py:171-175)
    const float xa_h[2] = {__shfl_sync(0xffffffffu, xa, (lane & ~3) | 0),
                           __shfl_sync(0xffffffffu, xa, (lane & ~3) | 1)};
    // the final state enters the divergence test too
    auto dfold = [&](float d, float a, float b) {
        if constexpr (SC)
            return min_nan3(d, fmaf(-a, a, s.alpha), fmaf(-b, b, s.alpha));
        else
            return max_nan3(d, a * a, b * b);
    };
    auto dmerge = [&](float a, float b) {
        if constexpr (SC)
            return min_nan(a, b);
        else
            return max_nan(a, b);
    };
    float dvh[2] = {dmerge(dv[0][0], dv[0][1]), dmerge(dv[1][0], dv[1][1])};
    // own aux spin: its tracked value and its final state
    if constexpr (SC)
        dvh[hown] = min_nan(dvh[hown], min_nan(dva, fmaf(-xa, xa, s.alpha)));
    else
        dvh[hown] = max_nan(dvh[hown], max_nan(dva, xa * xa));
    uint64_t pos[2], neg[2];
    bool dflag[2];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        float d = dvh[h];
        uint64_t pm = 0, nm = 0;
        const int64_t row = rowh[h];
        // (PACK: a missing second problem's rows are not written)
        int8_t* sp = spins + (hval[h] ? row : rowh[0]) * Sg;
        const bool wr = hval[h];
#pragma unroll
        for (int n = 0; n < NT; ++n) {
            d = dfold(d, xA[h][n].x, xA[h][n].y);
            d = dfold(d, xB[h][n].x, xB[h][n].y);
            const int i = 8 * n + 2 * t;
            const int a0 = xA[h][n].x >= 0.f ? 1 : -1, a1 = xA[h][n].y >= 0.f ? 1 : -1;
            const int b0 = xB[h][n].x >= 0.f ? 1 : -1, b1 = xB[h][n].y >= 0.f ? 1 : -1;
            if constexpr (!PAD) {
                if (wr) {
                    sp[i] = (int8_t)a0;
                    sp[i + 1] = (int8_t)a1;
                    sp[N + i] = (int8_t)b0;
                    sp[N + i + 1] = (int8_t)b1;
                }
                pm |= (uint64_t)(a0 + b0 == 2) << i | (uint64_t)(a1 + b1 == 2) << (i + 1);
                nm |= (uint64_t)(a0 + b0 == -2) << i | (uint64_t)(a1 + b1 == -2) << (i + 1);
            } else {  // inert spins are neither stored nor part of the configuration
                if (i < nr) {
                    if (wr) {
                        sp[i] = (int8_t)a0;
                        sp[nr + i] = (int8_t)b0;
                    }
                    pm |= (uint64_t)(a0 + b0 == 2) << i;
                    nm |= (uint64_t)(a0 + b0 == -2) << i;
                }
                if (i + 1 < nr) {
                    if (wr) {
                        sp[i + 1] = (int8_t)a1;
                        sp[nr + i + 1] = (int8_t)b1;
                    }
                    pm |= (uint64_t)(a1 + b1 == 2) << (i + 1);
                    nm |= (uint64_t)(a1 + b1 == -2) << (i + 1);
                }
            }
        }
        d = dmerge(d, __shfl_xor_sync(0xffffffffu, d, 1));
        d = dmerge(d, __shfl_xor_sync(0xffffffffu, d, 2));
        pm |= __shfl_xor_sync(0xffffffffu, pm, 1);
        pm |= __shfl_xor_sync(0xffffffffu, pm, 2);
        nm |= __shfl_xor_sync(0xffffffffu, nm, 1);
        nm |= __shfl_xor_sync(0xffffffffu, nm, 2);
        pos[h] = pm;
        neg[h] = nm;
        if (t == h && wr) sp[2 * nr] = xa >= 0.f ? 1 : -1;
        dflag[h] = SC ? !(d >= s.qthr) : !(d <= s.thr2);
        if (t == 0 && wr) diverged[row] = dflag[h] ? 1 : 0;
        if constexpr (PAD) {
            if (counting) {
                int c = cnt[h];
                c = min(c, __shfl_xor_sync(0xffffffffu, c, 1));
                c = min(c, __shfl_xor_sync(0xffffffffu, c, 2));
                const int a = PACK ? g : mt * 16 + g + 8 * h;
                if (t == 0 && a < s.b_out && wr) {
                    steps_out[probh[h] * s.b_out + a] = c;
                    mvms_out[probh[h] * s.b_out + a] = (c + s.f_mvm - 1) / s.f_mvm;
                }
            }
        }
    }
    if (screened) {
        // Selection screen: E + 2 tr G in FP32 from the tensor cores.  u =
        // s_A + s_B in {-2, 0, 2} is exact in f16, so two passes over the
        // staged hi/lo fragments give M = (-Ks G) u to ~2^-21 of sum|G|; the
        // anneals that can still be the argmin are re-evaluated in FP64.
        float2 u[2][NT];
#pragma unroll
        for (int h = 0; h < 2; ++h)
#pragma unroll
            for (int n = 0; n < NT; ++n)
                u[h][n] = make_float2((xA[h][n].x >= 0.f ? 1.f : -1.f) + (xB[h][n].x >= 0.f ? 1.f : -1.f),
                                      (xA[h][n].y >= 0.f ? 1.f : -1.f) + (xB[h][n].y >= 0.f ? 1.f : -1.f));
        float acc[NT][4];
#pragma unroll
        for (int n = 0; n < NT; ++n) acc[n][0] = acc[n][1] = acc[n][2] = acc[n][3] = 0.f;
        float keep[NT][2];
#pragma unroll
        for (int pq = 0; pq < NP; ++pq) {
            if (pq) {  // PACK: rows g keep the first problem's product
#pragma unroll
                for (int n = 0; n < NT; ++n) {
                    keep[n][0] = acc[n][0];
                    keep[n][1] = acc[n][1];
                    acc[n][0] = acc[n][1] = acc[n][2] = acc[n][3] = 0.f;
                }
            }
#pragma unroll
            for (int kt = 0; kt < KT; ++kt) {
                uint32_t a[4];
                a[0] = h2_bits(__float22half2_rn(u[0][2 * kt]));
                a[1] = h2_bits(__float22half2_rn(u[1][2 * kt]));
                a[2] = 2 * kt + 1 < NT ? h2_bits(__float22half2_rn(u[0][2 * kt + 1])) : 0u;
                a[3] = 2 * kt + 1 < NT ? h2_bits(__float22half2_rn(u[1][2 * kt + 1])) : 0u;
#pragma unroll
                for (int n = 0; n < NT; ++n) {
                    const uint4 f = frag[pq * L::kFragF4 + (kt * NT + n) * 32 + lane];
                    mma_f16(acc[n], a, f.z, f.w);
                    mma_f16(acc[n], a, f.x, f.y);
                }
            }
        }
        if constexpr (PACK) {
#pragma unroll
            for (int n = 0; n < NT; ++n) {
                acc[n][0] = keep[n][0];
                acc[n][1] = keep[n][1];
            }
        }
        // unscaled FP32-screen energies (without -2 tr G) of rows g, g+8
        double es[2];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            float q = 0.f, l = 0.f;
#pragma unroll
            for (int n = 0; n < NT; ++n) {
                q = fmaf(u[h][n].x, acc[n][2 * h], q);
                q = fmaf(u[h][n].y, acc[n][2 * h + 1], q);
                l = fmaf(nkb(h, n).x, u[h][n].x, l);
                l = fmaf(nkb(h, n).y, u[h][n].y, l);
            }
            float e = fmaf(xa_h[h] >= 0.f ? 2.f : -2.f, l, q);  // -Ks (u'Gu + 2 s_aux b'u)
            e += __shfl_xor_sync(0xffffffffu, e, 1);
            e += __shfl_xor_sync(0xffffffffu, e, 2);
            // padded rows (>= b_valid) never enter the selection
            // (a zero coupling scale leaves no screen: every survivor is a candidate)
            const double Kh = Ksq[PACK ? h : 0];
            es[h] = (dflag[h] || (PACK ? g : mt * 16 + g + 8 * h) >= s.b_valid) ? INFINITY
                    : (Kh > 0.0 ? (double)e * (-1.0 / Kh) : 0.0);
        }
        // tile minimum over survivors (PACK: per problem); candidates within
        // 2 x 2^-12 mag of it (the screen error is < 2^-13 mag, see launch_anneal_fast)
        const double* magp = reinterpret_cast<const double*>(frag + L::kKgF4 - 1);
        double lim[2];
        if constexpr (PACK) {
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                double m = es[h];
#pragma unroll
                for (int o = 4; o < 32; o <<= 1) m = fmin(m, __shfl_xor_sync(0xffffffffu, m, o));
                lim[h] = m + 0x1p-11 * magp[h];
            }
        } else {
            double m = fmin(es[0], es[1]);
#pragma unroll
            for (int o = 4; o < 32; o <<= 1) m = fmin(m, __shfl_xor_sync(0xffffffffu, m, o));
            lim[0] = lim[1] = m + 0x1p-11 * magp[0];
        }
        // lane 4g + h stands for row g + 8h (h < 2)
        const int hs = t & 1;
        const uint64_t my_pos = pos[hs], my_neg = neg[hs];
        const bool my_aux = xa >= 0.f;  // aux of row g + 8 hown, hown == hs
        const bool my_cand = t < 2 && es[hs] <= lim[hs];
        unsigned cand = __ballot_sync(0xffffffffu, my_cand);
        double my_e = INFINITY;
        double* w = reinterpret_cast<double*>(frag);  // fragments are consumed
        __syncwarp();
        double trq[NP];
#pragma unroll
        for (int q = 0; q < NP; ++q) {
            double tr = 0.0;
            for (int i = lane; i < nr; i += 32) tr += Gq[q][(int64_t)i * nr + i];
            trq[q] = warp_sum(tr);
        }
        while (cand) {
            const int l = __ffs(cand) - 1;
            const uint64_t cp = __shfl_sync(0xffffffffu, my_pos, l);
            const uint64_t cn = __shfl_sync(0xffffffffu, my_neg, l);
            const bool cax = __shfl_sync(0xffffffffu, my_aux, l);
            const int ch = PACK ? (l & 1) : 0;  // the candidate's problem
            const double* G = Gq[ch];
            const double* bv_p = bq[ch];
            const double tr = trq[ch];
            // E = u'Gu - 2 tr G + 2 s_aux b'u with u = 2 w (solver.py:171-175);
            // lane i sums row i through column i of the symmetric G
            for (int j = lane; j < N; j += 32)  // (inert spins: w = 0)
                w[j] = (double)((int)((cp >> j) & 1u) - (int)((cn >> j) & 1u));
            __syncwarp();
            double q = 0.0, li = 0.0;
            for (int i = lane; i < nr; i += 32) {
                double gu[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
                for (int j = 0; j < N; j += 4)
#pragma unroll
                    for (int r = 0; r < 4; ++r)
                        if (!PAD || j + r < nr)
                            gu[r] = fma(__ldg(G + (int64_t)(j + r) * nr + i), w[j + r], gu[r]);
                q = fma(w[i], (gu[0] + gu[1]) + (gu[2] + gu[3]), q);
                li = fma(bv_p[i], w[i], li);
            }
            __syncwarp();
            q = warp_sum(q);
            li = warp_sum(li);
            const double e = (4.0 * q - 2.0 * tr) + (cax ? 4.0 : -4.0) * li;
            // identical configurations (of the same problem) have identical energies
            const bool same = my_cand && my_pos == cp && my_neg == cn && my_aux == cax &&
                              (!PACK || hs == ch);
            if (same) my_e = e;
            cand &= ~__ballot_sync(0xffffffffu, same);
        }
        if (t < 2 && hval[t]) energies[rowh[t]] = my_e;
        return;
    }
    if constexpr (PACK) {
        // FP64 energies, PACK: row half h against its own problem's G, b
        double rs[2][2 * NT];
#pragma unroll
        for (int k = 0; k < 2 * NT; ++k) rs[0][k] = rs[1][k] = 0.0;
        for (int j = 0; j < nr; ++j) {
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const double sj = (double)((int)((pos[h] >> j) & 1u) - (int)((neg[h] >> j) & 1u));
                const double* Gj = Gq[h] + (int64_t)j * nr + 2 * t;
#pragma unroll
                for (int n = 0; n < NT; ++n) {
                    const int c = 8 * n + 2 * t;
                    const double2 gv = !PAD ? __ldg(reinterpret_cast<const double2*>(Gj + 8 * n))
                                            : make_double2(c < nr ? __ldg(Gj + 8 * n) : 0.0,
                                                           c + 1 < nr ? __ldg(Gj + 8 * n + 1) : 0.0);
                    rs[h][2 * n] = fma(gv.x, sj, rs[h][2 * n]);
                    rs[h][2 * n + 1] = fma(gv.y, sj, rs[h][2 * n + 1]);
                }
            }
        }
        double quad[2] = {0.0, 0.0}, lin[2] = {0.0, 0.0}, trh[2] = {0.0, 0.0};
#pragma unroll
        for (int n = 0; n < NT; ++n) {
#pragma unroll
            for (int dl = 0; dl < 2; ++dl) {
                const int i = 8 * n + 2 * t + dl;
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const double si = (double)((int)((pos[h] >> i) & 1u) - (int)((neg[h] >> i) & 1u));
                    quad[h] = fma(si, rs[h][2 * n + dl], quad[h]);
                    if (!PAD || i < nr) {
                        lin[h] = fma(bq[h][i], si, lin[h]);
                        trh[h] += Gq[h][(int64_t)i * nr + i];
                    }
                }
            }
        }
#pragma unroll
        for (int o = 1; o <= 2; o <<= 1)
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                quad[h] += __shfl_xor_sync(0xffffffffu, quad[h], o);
                lin[h] += __shfl_xor_sync(0xffffffffu, lin[h], o);
                trh[h] += __shfl_xor_sync(0xffffffffu, trh[h], o);
            }
        if (t < 2 && hval[t]) {
            const int h = t;
            const double aux = xa_h[h] >= 0.f ? 1.0 : -1.0;
            energies[rowh[h]] = (4.0 * quad[h] - 2.0 * trh[h]) + 4.0 * aux * lin[h];
        }
        return;
    }
    // FP64 energies.  Row sums use G's symmetry: sum_j s_j G[j][i] reads row j
    // at this lane's columns i = 8n+2t+{0,1} (16-byte loads), with s_j decoded
    // once per j for both anneals.
    const double* bg = bv_p;
    double rs[2][2 * NT];
#pragma unroll
    for (int k = 0; k < 2 * NT; ++k) rs[0][k] = rs[1][k] = 0.0;
    for (int j = 0; j < nr; ++j) {
        const double s0 = (double)((int)((pos[0] >> j) & 1u) - (int)((neg[0] >> j) & 1u));
        const double s1 = (double)((int)((pos[1] >> j) & 1u) - (int)((neg[1] >> j) & 1u));
        const double* Gj = G + (int64_t)j * nr + 2 * t;
#pragma unroll
        for (int n = 0; n < NT; ++n) {
            // (PAD: rows of odd length are not 16-byte aligned; inert columns read 0)
            const int c = 8 * n + 2 * t;
            const double2 gv = !PAD ? __ldg(reinterpret_cast<const double2*>(Gj + 8 * n))
                                    : make_double2(c < nr ? __ldg(Gj + 8 * n) : 0.0,
                                                   c + 1 < nr ? __ldg(Gj + 8 * n + 1) : 0.0);
            rs[0][2 * n] = fma(gv.x, s0, rs[0][2 * n]);
            rs[0][2 * n + 1] = fma(gv.y, s0, rs[0][2 * n + 1]);
            rs[1][2 * n] = fma(gv.x, s1, rs[1][2 * n]);
            rs[1][2 * n + 1] = fma(gv.y, s1, rs[1][2 * n + 1]);
        }
    }
    double quad[2] = {0.0, 0.0}, lin[2] = {0.0, 0.0}, tr = 0.0;
#pragma unroll
    for (int n = 0; n < NT; ++n) {
#pragma unroll
        for (int dl = 0; dl < 2; ++dl) {
            const int i = 8 * n + 2 * t + dl;
            const double si0 = (double)((int)((pos[0] >> i) & 1u) - (int)((neg[0] >> i) & 1u));
            const double si1 = (double)((int)((pos[1] >> i) & 1u) - (int)((neg[1] >> i) & 1u));
            quad[0] = fma(si0, rs[0][2 * n + dl], quad[0]);
            quad[1] = fma(si1, rs[1][2 * n + dl], quad[1]);
            if (!PAD || i < nr) {
                const double bi = bg[i];
                lin[0] = fma(bi, si0, lin[0]);
                lin[1] = fma(bi, si1, lin[1]);
                tr += G[(int64_t)i * nr + i];
            }
        }
    }
#pragma unroll
    for (int o = 1; o <= 2; o <<= 1) {
        quad[0] += __shfl_xor_sync(0xffffffffu, quad[0], o);
        quad[1] += __shfl_xor_sync(0xffffffffu, quad[1], o);
        lin[0] += __shfl_xor_sync(0xffffffffu, lin[0], o);
        lin[1] += __shfl_xor_sync(0xffffffffu, lin[1], o);
        tr += __shfl_xor_sync(0xffffffffu, tr, o);
    }
    if (t < 2) {
        const int h = t;
        const double aux = xa_h[h] >= 0.f ? 1.0 : -1.0;
        energies[rowh[h]] = (4.0 * quad[h] - 2.0 * tr) + 4.0 * aux * lin[h];
    }
}

template <int NT, bool SPLIT, bool SAME_QR, bool PAD, bool PACK>
int launch_cfg(const double* G, const double* g, const double* b, const uint64_t* base_seed,
               const double* eps_p, int64_t n_tasks, int tiles, const FastScalars& fs,
               int8_t* spins, uint8_t* diverged, double* energies, bool screened, int n_rt,
               int64_t* steps, int64_t* mvms, cudaStream_t st) {
    const int64_t blocks = (n_tasks + kWarpsPerCta - 1) / kWarpsPerCta;
    IL_REQUIRE(blocks < (1ll << 31), "too many problems in one launch");
    const size_t smem = FastLayout<NT, PACK>::kWarpBytes;
    auto fn = k_anneal_fast<NT, SPLIT, SAME_QR, PAD, PACK>;
    IL_CHECK_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    IL_CHECK_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
    IL_LAUNCH(kProfAnneal, st, fn<<<(unsigned)blocks, kWarpsPerCta * 32, smem, st>>>(G, g, b, base_seed, eps_p, n_tasks, tiles,
                                                        fs, spins, diverged, energies, screened, n_rt, steps, mvms););
    IL_CHECK_CUDA(cudaGetLastError());
    return IL_OK;
}

template <int NT, bool PAD, bool PACK>
int launch_pad(const double* G, const double* g, const double* b, const uint64_t* base_seed,
               const double* eps_p, int64_t n_tasks, int tiles, const FastScalars& fs, bool split,
               bool same_qr, int8_t* spins, uint8_t* diverged, double* energies, bool screened,
               int n_rt, int64_t* steps, int64_t* mvms, cudaStream_t st) {
#define IL_CFG(SP, SQ)                                                                                  \
    launch_cfg<NT, SP, SQ, PAD, PACK>(G, g, b, base_seed, eps_p, n_tasks, tiles, fs, spins, diverged,   \
                                      energies, screened, n_rt, steps, mvms, st)
    if (split) return same_qr ? IL_CFG(true, true) : IL_CFG(true, false);
    return same_qr ? IL_CFG(false, true) : IL_CFG(false, false);
#undef IL_CFG
}

template <int NT>
int launch_nt(const double* G, const double* g, const double* b, const uint64_t* base_seed,
              const double* eps_p, int64_t P, int B, const FastScalars& fs, bool split,
              bool same_qr, int8_t* spins, uint8_t* diverged, double* energies, bool screened,
              int n_rt, int64_t* steps, int64_t* mvms, cudaStream_t st) {
    const bool pad = !(n_rt == 8 * NT && steps == nullptr);
    if (B == 8) {  // two 8-anneal problems per warp
        const int64_t n_tasks = (P + 1) / 2;
        return pad ? launch_pad<NT, true, true>(G, g, b, base_seed, eps_p, n_tasks, 1, fs, split, same_qr,
                                                spins, diverged, energies, screened, n_rt, steps, mvms, st)
                   : launch_pad<NT, false, true>(G, g, b, base_seed, eps_p, n_tasks, 1, fs, split, same_qr,
                                                 spins, diverged, energies, screened, n_rt, steps, mvms, st);
    }
    const int tiles = B / 16;
    const int64_t n_tasks = P * tiles;
    return pad ? launch_pad<NT, true, false>(G, g, b, base_seed, eps_p, n_tasks, tiles, fs, split, same_qr,
                                             spins, diverged, energies, screened, n_rt, steps, mvms, st)
               : launch_pad<NT, false, false>(G, g, b, base_seed, eps_p, n_tasks, tiles, fs, split, same_qr,
                                              spins, diverged, energies, screened, n_rt, steps, mvms, st);
}

}  // namespace fast_impl

// per-layout entry points (anneal_fast_nt<k>.cu)
#define IL_FAST_NT_DECL(k)                                                                           \
    int launch_fast_nt##k(const double* G, const double* g, const double* b,                        \
                          const uint64_t* base_seed, const double* eps_p, int64_t P, int B,         \
                          const fastk::FastScalars& fs, bool split, bool same_qr, int8_t* spins,    \
                          uint8_t* diverged, double* energies, bool screened, int n_rt,             \
                          int64_t* steps, int64_t* mvms, cudaStream_t st)
IL_FAST_NT_DECL(1);
IL_FAST_NT_DECL(2);
IL_FAST_NT_DECL(3);
IL_FAST_NT_DECL(4);
IL_FAST_NT_DECL(5);
IL_FAST_NT_DECL(6);
IL_FAST_NT_DECL(7);
IL_FAST_NT_DECL(8);

}  // namespace il
