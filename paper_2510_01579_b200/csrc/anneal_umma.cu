// CIM-CAC anneal with the coupling product on the 5th-generation tensor
// cores (tcgen05.mma, accumulator in TMEM).  Same dynamics, state layout and
// outputs as k_anneal_fast (anneal_fast.cu); only the refresh differs.
//
// Why: the legacy mma.sync refresh costs 24 HMMA.16816 per warp and period,
// and each one blocks the warp scheduler for ~5 cycles even when independent
// FP32 work is available (tools/microbench/overlap.cu), so the tensor work
// adds to the FP32-pipe-bound Euler work instead of hiding under it.  A
// tcgen05.mma is issued by one thread for the whole CTA and runs
// asynchronously: the CTA's other warps, and the other CTAs of the SM, keep
// the FP32 pipes busy while it runs.
//
// Mapping (CTA = 4 warps, 64 anneal rows; warp q owns rows 16q..16q+15):
//   D[64 x NB] = A[64 x K] * B[K x NB]  (kind::f16, fp32 accumulate, M = 64)
//   A row 16q + r: v = x1 + x2 of the warp's anneal r (f16 hi or lo part),
//   written by its owner thread in the canonical K-major core-matrix layout;
//   B: the CTA's problems side by side (NB = problems x N columns), -Ks G per
//   problem in f16 hi/lo, staged once.  Rows of one problem times the other
//   problems' columns are not used (M = 64 is the smallest 1-CTA tile).
//   M = 64 places row m in TMEM lane (m % 16) + 32 (m / 16): warp q reads its
//   16 rows, its own problem's columns, with tcgen05.ld.16x256b -- exactly
//   the mma.sync accumulator fragment, so the Euler update is unchanged.
//   FP32 mode: 3 passes (hi.hi + lo.hi + hi.lo) as in anneal_fast.cu.
// Per refresh: every warp stores its A rows, fence.proxy.async, CTA barrier,
// thread 0 issues the MMAs, one column block per problem, each committed to
// its own mbarrier; every warp waits on its block and loads its fragment.
//
// Measured (16x16 16-QAM slot, B200): 4.70 ms against 4.53 ms for the
// mma.sync kernel, so it is not the default (ISINGLINK_UMMA=1 selects it).
// With 32 anneals per problem the product per problem is 32 x 32 x 32, below
// the smallest 1-CTA tcgen05 tile (M = 64, itself at half rate): the CTA
// tile computes 2x the useful MACs, and the barrier plus the exposed MMA
// latency per refresh cost more than the HMMA issue slots they free.  The
// per-warp variant (IL_UMMA_PERWARP, no barrier, 4x the MACs) takes 5.67 ms.
#include <cuda_fp16.h>

#include "il_anneal.cuh"
#include "il_internal.cuh"
#include "rng_numpy.cuh"

namespace il {

namespace {
using namespace fastk;

constexpr int kUWarps = 4;
#ifndef IL_UMMA_PERWARP  // each warp issues its own M = 64 product (no CTA barrier)
#define IL_UMMA_PERWARP 0
#endif

// ---- tcgen05 / TMEM primitives ---------------------------------------------
IL_D void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
IL_D void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
IL_D void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

// Shared-memory matrix descriptor: canonical K-major layout without swizzle;
// core matrices of 8 rows x 16 bytes, `lbo` bytes between the two K-halves of
// one 16-wide K step, `sbo` bytes between 8-row groups.
IL_D uint64_t smem_desc(const void* p, uint32_t lbo, uint32_t sbo) {
    uint64_t d = (uint64_t)((smem_u32(p) & 0x3FFFFu) >> 4);
    d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
    d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
    d |= (uint64_t)1 << 46;  // descriptor version (sm_100)
    return d;                // base offset 0, SWIZZLE_NONE
}

// Instruction descriptor: kind::f16, A = B = f16, D = f32, both K-major.
constexpr uint32_t idesc_f16(int M, int N) {
    return (1u << 4) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

IL_D void umma_f16(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
        " tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(d_tmem),
        "l"(a), "l"(b), "r"(idesc), "r"(acc)
        : "memory");
}
IL_D void umma_commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                     smem_u32(bar))
                 : "memory");
}
// 16 TMEM lanes x 8 columns: the m16n8 accumulator fragment of this lane
IL_D void tmem_ld_frag(uint32_t taddr, float (&r)[4]) {
    asm volatile("tcgen05.ld.sync.aligned.16x256b.x1.b32 {%0, %1, %2, %3}, [%4];"
                 : "=f"(r[0]), "=f"(r[1]), "=f"(r[2]), "=f"(r[3])
                 : "r"(taddr)
                 : "memory");
}
IL_D void tmem_ld_wait() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

// mbarrier wait with a watchdog: a lost arrive traps instead of hanging
IL_D void mbar_wait_guard(uint64_t* bar, uint32_t parity) {
    uint32_t done = 0, spins = 0;
    while (true) {
        asm volatile(
            "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
            " selp.u32 %0, 1, 0, p;\n}\n"
            : "=r"(done)
            : "r"(smem_u32(bar)), "r"(parity)
            : "memory");
        if (done) return;
        if (++spins > (1u << 26)) __trap();
    }
}

template <int NT>
struct ULayout {
    static constexpr int N = 8 * NT;
    static constexpr int S = 2 * N + 1;
    static constexpr int KT = (NT + 1) / 2;  // 16-wide K steps
    static constexpr int KP = 16 * KT;       // padded K
    static constexpr int M = 64;
    // canonical K-major operand: chunk c (8 K values) of row group r at
    // (c * rows / 8 + r) * 128 bytes, row i of the group at + 16 i
    static constexpr uint32_t kABytes = M * KP * 2;  // one f16 part of A
    static constexpr int kX0Floats = 16 * S;
    static constexpr size_t kHdr = 128;  // mbarriers, TMEM address, per-warp scalars
    static size_t smem(int nb) {
        return kHdr + 2 * (size_t)kABytes + 2 * (size_t)nb * KP * 2 +
               (size_t)kUWarps * ((kX0Floats * 4 + 15) / 16 * 16);
    }
};

// byte offset of element (row, k) of a K-major operand with `rows` rows
IL_D uint32_t kmaj_off(int row, int k, int rows) {
    return (uint32_t)(((k >> 3) * (rows >> 3) + (row >> 3)) * 128 + (row & 7) * 16 + (k & 7) * 2);
}

template <int NT, bool SPLIT, bool SAME_QR>
__global__ void __launch_bounds__(kUWarps * 32, NT <= 2 ? 4 : (NT <= 4 ? 3 : 1))
k_anneal_umma(const double* __restrict__ Gall, const double* __restrict__ gall,
              const double* __restrict__ ball, const uint64_t* __restrict__ base_seed,
              const double* __restrict__ eps_p, int64_t n_tasks, int64_t P, int tiles_per_prob,
              int nb, int tmem_cols, FastScalars s, int8_t* __restrict__ spins,
              uint8_t* __restrict__ diverged, double* __restrict__ energies, bool screened) {
    using L = ULayout<NT>;
    constexpr int N = L::N;
    constexpr int S = L::S;
    constexpr int KT = L::KT;
    constexpr int KP = L::KP;
    extern __shared__ __align__(128) uint8_t smem[];
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem);          // [4] D ready, per warp
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + 32);
    double* warp_scal = reinterpret_cast<double*>(smem + 64);    // [4]
    uint8_t* A_hi = smem + L::kHdr;
    uint8_t* A_lo = A_hi + L::kABytes;
    uint8_t* B_hi = A_lo + L::kABytes;
    uint8_t* B_lo = B_hi + (size_t)nb * KP * 2;
    float* x0_all = reinterpret_cast<float*>(B_lo + (size_t)nb * KP * 2);

    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t task0 = (int64_t)blockIdx.x * kUWarps;
    const int64_t task = task0 + warp;
    const bool valid = task < n_tasks;
    // warps past the end run on the last task (their outputs are dropped):
    // every warp takes part in the CTA's MMAs and barriers
    const int64_t tsk = valid ? task : n_tasks - 1;
    const int64_t prob = tsk / tiles_per_prob;
    const int mt = (int)(tsk % tiles_per_prob);
    const int pslot = warp / tiles_per_prob;  // problem slot of this warp in the CTA
    const int B = tiles_per_prob * 16;
    const int g = lane >> 2, t = lane & 3;
    const int hown = t & 1;
    const double* G = Gall + prob * (int64_t)N * N;

    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                         smem_u32(tmem_slot)),
                     "r"(tmem_cols)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    if (threadIdx.x >= 32 && threadIdx.x < 32 + kUWarps) {
        mbar_init(bars + threadIdx.x - 32, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }

    // ---- initial states: replayed NumPy streams, 2 lanes per anneal ---------
    float* x0s = x0_all + warp * ((L::kX0Floats + 3) / 4 * 4);
    {
        const int al = lane & 15, part = lane >> 4;
        const int a = mt * 16 + al;
        Pcg64 rng;
        rng.seed_from(derive_seed2(base_seed[prob], (uint64_t)a));
        constexpr int S0 = (S + 1) / 2;
        if (part) rng.state = add128(mul128(rng.state, s.jump_mult[3]), mul128(rng.inc, s.jump_add[3]));
        const int i0 = part ? S0 : 0, i1 = part ? S : S0;
        for (int i = i0; i < i1; ++i) x0s[al * S + i] = (float)rng.uniform(s.x0_lo, s.x0_range);
    }

    // ---- per-problem scale 2^sc for -K*G (and the screen bound) --------------
    const double K = s.dt * eps_p[prob];
    double gmax = 0.0, mag = 0.0;
#pragma unroll 4
    for (int i = lane; i < N * N; i += 32) {
        const double v = fabs(__ldg(G + i));
        gmax = fmax(gmax, v);
        mag += v;
    }
    for (int i = lane; i < N; i += 32) mag += fabs(ball[prob * N + i]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) gmax = fmax(gmax, __shfl_xor_sync(0xffffffffu, gmax, o));
    mag = warp_sum(mag);
    if (lane == 0) warp_scal[warp] = mag;
    int ex = 0;
    frexp(K * gmax, &ex);
    const int sc = (K * gmax > 0.0) ? 8 - ex : 0;
    const double Ks = ldexp(K, sc);
    const float e_init = ldexpf(1.0f, -sc);
    const float e_floor = ldexpf(s.e_floor, -sc);

    // ---- stage this warp's share of the B columns: problem pslot, spin
    //      columns c0 .. c0 + N / tiles - 1, all KP rows (K beyond N is zero)
    {
        const int per = N / tiles_per_prob;
        const int c0 = mt * per;
        const int col_base = pslot * N;
        for (int idx = lane; idx < per * (KP / 2); idx += 32) {
            const int c = c0 + idx % per, k = 2 * (idx / per);
            float f0 = 0.f, f1 = 0.f;
            if (k < N) f0 = (float)(-Ks * __ldg(G + (int64_t)k * N + c));
            if (k + 1 < N) f1 = (float)(-Ks * __ldg(G + (int64_t)(k + 1) * N + c));
            uint32_t hi, lo;
            split_h2(make_float2(f0, f1), hi, lo);
            const uint32_t off = kmaj_off(col_base + c, k, nb);
            *reinterpret_cast<uint32_t*>(B_hi + off) = hi;
            *reinterpret_cast<uint32_t*>(B_lo + off) = lo;
        }
        fence_async_smem();
    }

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
            eA[h][n] = eB[h][n] = make_float2(e_init, e_init);
            CA[h][n] = CB[h][n] = make_float2(0.f, 0.f);
        }
    }
    float xa = x0s[(g + 8 * hown) * S + 2 * N], ea = e_init, Ca = 0.f, dva = 0.f;
    float dv[2][2] = {{0.f, 0.f}, {0.f, 0.f}};
    float e_lb = e_init;
    float2 Kg[NT], nKb[NT];
#pragma unroll
    for (int n = 0; n < NT; ++n) {
        const int i = 8 * n + 2 * t;
        Kg[n] = make_float2((float)(Ks * gall[prob * N + i]), (float)(Ks * gall[prob * N + i + 1]));
        nKb[n] = make_float2((float)(-Ks * ball[prob * N + i]), (float)(-Ks * ball[prob * N + i + 1]));
    }

    // TMEM base address (written by warp 0's alloc) and barrier init visible
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
#if IL_UMMA_PERWARP
    // Each warp issues its own product: all 64 A rows (the other warps' rows
    // are don't-care for this warp's output rows) times its problem's N
    // columns of B into a private D region (TMEM columns warp * N ..), so no
    // CTA-wide barrier is needed -- at 4x the tensor work of the useful rows.
    const uint32_t dcol = (uint32_t)(warp * N);
    uint64_t* dbar = bars + warp;
#else
    // One product per CTA refresh over all nb columns, issued by thread 0
    // after a CTA barrier (one instruction per K step and pass: splitting it
    // into per-problem column blocks, each committed on its own, measured
    // 5.70 ms -- small-N tcgen05 instructions cost about as much as N = 64).
    const uint32_t dcol = (uint32_t)(pslot * N);
    uint64_t* dbar = bars;
#endif
    // D row m sits in TMEM lane (m % 16) + 32 (m / 16): this warp's rows
    // 16 warp .. +15 are in its own lane quadrant
    const uint32_t tacc = tmem + ((uint32_t)(32 * warp) << 16) + dcol;
    const uint64_t adh = smem_desc(A_hi, 8 * 128, 128), adl = smem_desc(A_lo, 8 * 128, 128);
    uint32_t phase = 0;

    // the MMAs for B columns ps N .. ps N + ncols - 1 into D columns dc ..
    auto issue_block = [&](int ps, uint32_t dc, int ncols, int passes) {
        const uint32_t idesc = idesc_f16(64, ncols);
        const uint32_t bcol = (uint32_t)(ps * N / 8) * 128;  // row group ps N / 8 of B
        const uint64_t bdh = smem_desc(B_hi + bcol, (uint32_t)nb * 16, 128);
        const uint64_t bdl = smem_desc(B_lo + bcol, (uint32_t)nb * 16, 128);
        const uint32_t d = tmem + dc;
        uint32_t first = 0;
#pragma unroll
        for (int kt = 0; kt < KT; ++kt) {
            // K step kt covers core-matrix chunks 2kt, 2kt+1: 2 x 1024 bytes
            // into A (64 rows), 2 x nb x 16 bytes into B
            const uint64_t ao = (uint64_t)((2 * kt * 8 * 128) >> 4);
            const uint64_t bo = (uint64_t)((2 * kt * nb * 16) >> 4);
            umma_f16(d, adh + ao, bdh + bo, idesc, first);
            first = 1;
            if (passes >= 2) umma_f16(d, adh + ao, bdl + bo, idesc, 1);
            if (passes >= 3) umma_f16(d, adl + ao, bdh + bo, idesc, 1);
        }
    };
    auto warp_product = [&](int passes, float (&acc)[NT][4]) {
        fence_async_smem();
        tc_fence_before();
#if IL_UMMA_PERWARP
        __syncwarp();
        if (lane == 0) {
            tc_fence_after();
            issue_block(pslot, dcol, N, passes);
            umma_commit(dbar);
        }
        __syncwarp();
#else
        asm volatile("bar.sync 1, 128;" ::: "memory");
        if (threadIdx.x == 0) {
            tc_fence_after();
            issue_block(0, 0u, nb, passes);
            umma_commit(dbar);
        }
#endif
        mbar_wait_guard(dbar, phase);
        phase ^= 1u;
        tc_fence_after();
#pragma unroll
        for (int n = 0; n < NT; ++n) tmem_ld_frag(tacc + 8 * n, acc[n]);
        tmem_ld_wait();
    };
    // A row of anneal r = g + 8h of this warp: 16 warp + r
    auto store_a = [&](uint8_t* base, int h, int n, uint32_t v) {
        *reinterpret_cast<uint32_t*>(base + kmaj_off(16 * warp + g + 8 * h, 8 * n + 2 * t, 64)) = v;
    };
    if constexpr (KP > N) {  // zero K padding columns of A once (N = 8 NT, NT odd)
        for (int h = 0; h < 2; ++h) {
            store_a(A_hi, h, NT, 0u);
            store_a(A_lo, h, NT, 0u);
        }
    }

    int until_refresh = 0;
    for (int step = 0; step < s.n_steps; ++step) {
        if (until_refresh == 0) {
            until_refresh = s.f_mvm;
            float pb[2];
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                float2 p2 = make_float2(0.f, 0.f);
#pragma unroll
                for (int n = 0; n < NT; ++n) {
                    const float2 v = __fadd2_rn(xA[h][n], xB[h][n]);
                    p2 = __ffma2_rn(nKb[n], v, p2);
                    uint32_t hi, lo;
                    split_h2(v, hi, lo);
                    store_a(A_hi, h, n, hi);
                    if (SPLIT) store_a(A_lo, h, n, lo);
                }
                pb[h] = p2.x + p2.y;
            }
            const float xa0 = __shfl_sync(0xffffffffu, xa, (lane & ~3) | 0);
            const float xa1 = __shfl_sync(0xffffffffu, xa, (lane & ~3) | 1);
            {
                const float mine = hown ? pb[1] : pb[0];
                const float other = hown ? pb[0] : pb[1];
                float tot = mine + __shfl_xor_sync(0xffffffffu, other, 1);
                tot += __shfl_xor_sync(0xffffffffu, tot, 2);
                Ca = tot;
            }
            float acc[NT][4];
            warp_product(SPLIT ? 3 : 1, acc);
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const float xah = h ? xa1 : xa0;
#pragma unroll
                for (int n = 0; n < NT; ++n) {
                    const float2 m2 = make_float2(acc[n][2 * h], acc[n][2 * h + 1]);
                    const float2 u2 = __ffma2_rn(nKb[n], make_float2(xah, xah), m2);
                    CA[h][n] = __ffma2_rn(Kg[n], xA[h][n], u2);
                    CB[h][n] = __ffma2_rn(Kg[n], xB[h][n], u2);
                }
            }
        }
#pragma unroll
        for (int h = 0; h < 2; ++h) {
#pragma unroll
            for (int n = 0; n < NT; ++n) {
                euler_pair<SAME_QR>(xA[h][n], eA[h][n], CA[h][n], s, e_floor, dv[h][n & 1]);
                euler_pair<SAME_QR>(xB[h][n], eB[h][n], CB[h][n], s, e_floor, dv[h][n & 1]);
            }
        }
        {  // e floor through the per-thread lower bound (see anneal_fast.cu)
            const float dmax = max_nan3(max_nan(dv[0][0], dv[0][1]), dv[1][0], dv[1][1]);
            const float r_lb = SAME_QR ? fmaf(s.ndt, dmax, s.alpha) : fmaf(s.ndtz, dmax, s.beta);
            const float nxt = e_lb * r_lb;
            if (nxt >= e_floor) {
                e_lb = nxt;
            } else {
#pragma unroll
                for (int h = 0; h < 2; ++h)
#pragma unroll
                    for (int n = 0; n < NT; ++n) {
                        eA[h][n] = floor2(eA[h][n], e_floor);
                        eB[h][n] = floor2(eB[h][n], e_floor);
                    }
                e_lb = e_floor;
            }
        }
        euler_one<SAME_QR>(xa, ea, Ca, s, e_floor, dva);
        --until_refresh;
    }

    // ---- epilogue: divergence flags, spins ---------------------------------
    const float xa_h[2] = {__shfl_sync(0xffffffffu, xa, (lane & ~3) | 0),
                           __shfl_sync(0xffffffffu, xa, (lane & ~3) | 1)};
    float dvh[2] = {max_nan(dv[0][0], dv[0][1]), max_nan(dv[1][0], dv[1][1])};
    dvh[hown] = max_nan(dvh[hown], max_nan(dva, xa * xa));
    const int64_t row0 = prob * (int64_t)B + mt * 16;
    uint64_t pos[2], neg[2];
    bool dflag[2];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        float d = dvh[h];
        uint64_t pm = 0, nm = 0;
        const int64_t row = row0 + g + 8 * h;
        int8_t* sp = spins + row * S;
#pragma unroll
        for (int n = 0; n < NT; ++n) {
            d = max_nan3(d, xA[h][n].x * xA[h][n].x, xA[h][n].y * xA[h][n].y);
            d = max_nan3(d, xB[h][n].x * xB[h][n].x, xB[h][n].y * xB[h][n].y);
            const int i = 8 * n + 2 * t;
            const int a0 = xA[h][n].x >= 0.f ? 1 : -1, a1 = xA[h][n].y >= 0.f ? 1 : -1;
            const int b0 = xB[h][n].x >= 0.f ? 1 : -1, b1 = xB[h][n].y >= 0.f ? 1 : -1;
            if (valid) {
                sp[i] = (int8_t)a0;
                sp[i + 1] = (int8_t)a1;
                sp[N + i] = (int8_t)b0;
                sp[N + i + 1] = (int8_t)b1;
            }
            pm |= (uint64_t)(a0 + b0 == 2) << i | (uint64_t)(a1 + b1 == 2) << (i + 1);
            nm |= (uint64_t)(a0 + b0 == -2) << i | (uint64_t)(a1 + b1 == -2) << (i + 1);
        }
        d = max_nan(d, __shfl_xor_sync(0xffffffffu, d, 1));
        d = max_nan(d, __shfl_xor_sync(0xffffffffu, d, 2));
        pm |= __shfl_xor_sync(0xffffffffu, pm, 1);
        pm |= __shfl_xor_sync(0xffffffffu, pm, 2);
        nm |= __shfl_xor_sync(0xffffffffu, nm, 1);
        nm |= __shfl_xor_sync(0xffffffffu, nm, 2);
        pos[h] = pm;
        neg[h] = nm;
        dflag[h] = !(d <= s.thr2);
        if (valid && t == h) sp[2 * N] = xa >= 0.f ? 1 : -1;
        if (valid && t == 0) diverged[row] = dflag[h] ? 1 : 0;
    }

    double es[2] = {INFINITY, INFINITY};
    if (screened) {
        // FP32 screen on the tensor cores: u = s_A + s_B in {-2, 0, 2} (exact
        // in f16) against the hi and lo parts of B (see anneal_fast.cu)
        float2 u[2][NT];
#pragma unroll
        for (int h = 0; h < 2; ++h)
#pragma unroll
            for (int n = 0; n < NT; ++n) {
                u[h][n] = make_float2((xA[h][n].x >= 0.f ? 1.f : -1.f) + (xB[h][n].x >= 0.f ? 1.f : -1.f),
                                      (xA[h][n].y >= 0.f ? 1.f : -1.f) + (xB[h][n].y >= 0.f ? 1.f : -1.f));
                store_a(A_hi, h, n, h2_bits(__float22half2_rn(u[h][n])));
            }
        float acc[NT][4];
        warp_product(2, acc);
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            float q = 0.f, l = 0.f;
#pragma unroll
            for (int n = 0; n < NT; ++n) {
                q = fmaf(u[h][n].x, acc[n][2 * h], q);
                q = fmaf(u[h][n].y, acc[n][2 * h + 1], q);
                l = fmaf(nKb[n].x, u[h][n].x, l);
                l = fmaf(nKb[n].y, u[h][n].y, l);
            }
            float e = fmaf(xa_h[h] >= 0.f ? 2.f : -2.f, l, q);
            e += __shfl_xor_sync(0xffffffffu, e, 1);
            e += __shfl_xor_sync(0xffffffffu, e, 2);
            // (a zero coupling scale leaves no screen: every survivor is a candidate)
            es[h] = (dflag[h] || mt * 16 + g + 8 * h >= s.b_valid) ? INFINITY
                    : (Ks > 0.0 ? (double)e * (-1.0 / Ks) : 0.0);
        }
    }
    // TMEM is no longer needed by any warp
    tc_fence_before();
    __syncthreads();
    if (warp == 0) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                     "r"(tmem_cols)
                     : "memory");
    }
    if (!valid) return;

    const double* bg = ball + prob * N;
    if (screened) {
        // FP64 energies of the distinct configurations within the screen
        // bound of the tile minimum, +inf for the rest (anneal_fast.cu)
        double m = fmin(es[0], es[1]);
#pragma unroll
        for (int o = 4; o < 32; o <<= 1) m = fmin(m, __shfl_xor_sync(0xffffffffu, m, o));
        const double lim = m + 0x1p-11 * warp_scal[warp];
        const int hs = t & 1;
        const uint64_t my_pos = pos[hs], my_neg = neg[hs];
        const bool my_aux = xa >= 0.f;
        const bool my_cand = t < 2 && es[hs] <= lim;
        unsigned cand = __ballot_sync(0xffffffffu, my_cand);
        double my_e = INFINITY;
        double* w = reinterpret_cast<double*>(x0s);  // x0 staging is consumed
        double tr = 0.0;
        for (int i = lane; i < N; i += 32) tr += __ldg(G + (int64_t)i * N + i);
        tr = warp_sum(tr);
        while (cand) {
            const int l = __ffs(cand) - 1;
            const uint64_t cp = __shfl_sync(0xffffffffu, my_pos, l);
            const uint64_t cn = __shfl_sync(0xffffffffu, my_neg, l);
            const bool cax = __shfl_sync(0xffffffffu, my_aux, l);
            for (int j = lane; j < N; j += 32)
                w[j] = (double)((int)((cp >> j) & 1u) - (int)((cn >> j) & 1u));
            __syncwarp();
            double q = 0.0, li = 0.0;
            for (int i = lane; i < N; i += 32) {
                double gu[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
                for (int j = 0; j < N; j += 4)
#pragma unroll
                    for (int r = 0; r < 4; ++r)
                        gu[r] = fma(__ldg(G + (int64_t)(j + r) * N + i), w[j + r], gu[r]);
                q = fma(w[i], (gu[0] + gu[1]) + (gu[2] + gu[3]), q);
                li = fma(bg[i], w[i], li);
            }
            __syncwarp();
            q = warp_sum(q);
            li = warp_sum(li);
            const double e = (4.0 * q - 2.0 * tr) + (cax ? 4.0 : -4.0) * li;
            const bool same = my_cand && my_pos == cp && my_neg == cn && my_aux == cax;
            if (same) my_e = e;
            cand &= ~__ballot_sync(0xffffffffu, same);
        }
        if (t < 2) energies[row0 + g + 8 * t] = my_e;
        return;
    }
    // FP64 energies of every anneal (as anneal_fast.cu)
    double rs[2][2 * NT];
#pragma unroll
    for (int k = 0; k < 2 * NT; ++k) rs[0][k] = rs[1][k] = 0.0;
    for (int j = 0; j < N; ++j) {
        const double s0 = (double)((int)((pos[0] >> j) & 1u) - (int)((neg[0] >> j) & 1u));
        const double s1 = (double)((int)((pos[1] >> j) & 1u) - (int)((neg[1] >> j) & 1u));
        const double* Gj = G + (int64_t)j * N + 2 * t;
#pragma unroll
        for (int n = 0; n < NT; ++n) {
            const double2 gv = __ldg(reinterpret_cast<const double2*>(Gj + 8 * n));
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
            const double bi = __ldg(bg + i);
            lin[0] = fma(bi, si0, lin[0]);
            lin[1] = fma(bi, si1, lin[1]);
            tr += __ldg(G + (int64_t)i * N + i);
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
        energies[row0 + g + 8 * h] = (4.0 * quad[h] - 2.0 * tr) + 4.0 * aux * lin[h];
    }
}

template <int NT, bool SPLIT, bool SAME_QR>
int launch_u(const double* G, const double* g, const double* b, const uint64_t* base_seed,
             const double* eps_p, int64_t P, int tiles, const FastScalars& fs, int8_t* spins,
             uint8_t* diverged, double* energies, bool screened, cudaStream_t st) {
    constexpr int N = 8 * NT;
    const int64_t n_tasks = P * tiles;
    const int64_t blocks = (n_tasks + kUWarps - 1) / kUWarps;
    IL_REQUIRE(blocks < (1ll << 31), "too many problems in one launch");
    const int nb = (kUWarps / tiles) * N;  // B columns: problems per CTA x N
    int cols = 32;  // D: the CTA's columns, or one N-column region per warp
    while (cols < (IL_UMMA_PERWARP ? kUWarps * N : nb)) cols *= 2;
    const size_t smem = ULayout<NT>::smem(nb);
    auto fn = k_anneal_umma<NT, SPLIT, SAME_QR>;
    IL_CHECK_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    IL_LAUNCH(kProfAnneal, st,
              fn<<<(unsigned)blocks, kUWarps * 32, smem, st>>>(G, g, b, base_seed, eps_p, n_tasks, P,
                                                              tiles, nb, cols, fs, spins, diverged,
                                                              energies, screened););
    IL_CHECK_CUDA(cudaGetLastError());
    return IL_OK;
}

template <int NT>
int launch_u_nt(const double* G, const double* g, const double* b, const uint64_t* base_seed,
                const double* eps_p, int64_t P, int tiles, const FastScalars& fs, bool split,
                bool same_qr, int8_t* spins, uint8_t* diverged, double* energies, bool screened,
                cudaStream_t st) {
    if (split)
        return same_qr ? launch_u<NT, true, true>(G, g, b, base_seed, eps_p, P, tiles, fs, spins,
                                                  diverged, energies, screened, st)
                       : launch_u<NT, true, false>(G, g, b, base_seed, eps_p, P, tiles, fs, spins,
                                                   diverged, energies, screened, st);
    return same_qr ? launch_u<NT, false, true>(G, g, b, base_seed, eps_p, P, tiles, fs, spins,
                                               diverged, energies, screened, st)
                   : launch_u<NT, false, false>(G, g, b, base_seed, eps_p, P, tiles, fs, spins,
                                                diverged, energies, screened, st);
}

}  // namespace

bool umma_anneal_supported(int N, int B) {
    const int tiles = B / 16;
    if (B % 16 || !(tiles == 1 || tiles == 2 || tiles == 4)) return false;
    const int nb = (kUWarps / tiles) * N;
    return N % 8 == 0 && N >= 16 && N <= 64 && nb <= 256 && (N / 8) != 5 && (N / 8) != 7;
}

int launch_anneal_umma(const double* G, const double* g, const double* b,
                       const uint64_t* base_seed, const double* eps_p, int64_t P, int N, int B,
                       const void* fs_v, bool split, bool same_qr, int8_t* spins,
                       uint8_t* diverged, double* energies, bool screened, cudaStream_t st) {
    const FastScalars& fs = *static_cast<const FastScalars*>(fs_v);
    const int tiles = B / 16;
#define IL_UNT(k) \
    case k: return launch_u_nt<k>(G, g, b, base_seed, eps_p, P, tiles, fs, split, same_qr, spins, diverged, energies, screened, st)
    switch (N / 8) {
        IL_UNT(2);
        IL_UNT(3);
        IL_UNT(4);
        IL_UNT(6);
        IL_UNT(8);
#undef IL_UNT
        default:
            set_error("tcgen05 anneal kernel not instantiated for n_dim=%d", N);
            return IL_ERR_UNSUPPORTED;
    }
}

}  // namespace il
