// FP64-exact CIM-CAC anneal kernel.
//
// Reproduces the reference "ext" kernel (_kernel.pyx:16-102) bit for bit:
// same evaluation order (the Cython-generated C, _kernel.pyx:65-100), every
// multiply and add rounded separately (__dmul_rn/__dadd_rn/__dsub_rn: no FMA
// contraction), sequential j-order accumulation in the coupling product,
// halt-on-divergence with the state frozen at the halting step, sign(0)=+1.
//
// Mapping: one thread = one anneal, one warp = up to 32 anneals of the same
// problem; G, g_diag, b are staged once per CTA in shared memory and read as
// warp-wide broadcasts; the per-anneal state x, e, coupling, v lives in
// shared memory as [index][lane] so every access is conflict-free.
//
// Used (a) as the drop-in `run_anneals` plugin (x0 supplied by the caller)
// and (b) inside the batched pipelines in IL_PREC_FP64_EXACT mode, where x0
// is generated on the device from the replayed NumPy streams.
#include "il_internal.cuh"
#include "rng_numpy.cuh"
#include "rng_philox.cuh"

namespace il {

namespace {

constexpr int kLanes = 32;
#ifndef IL_EXACT_WARPS  // warps per 32-anneal chunk in the FP64-exact kernel
#define IL_EXACT_WARPS 4
#endif

__device__ __forceinline__ double dmul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double dadd(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double dsub(double a, double b) { return __dsub_rn(a, b); }

__global__ void __launch_bounds__(kLanes)
k_anneal_exact(const double* __restrict__ Gall, const double* __restrict__ gall,
               const double* __restrict__ ball, const double* __restrict__ x0all,
               const uint64_t* __restrict__ base_seed, const double* __restrict__ eps_p,
               int64_t P, int N, int B, int chunks, AnnealScalars s, int8_t* __restrict__ spins,
               uint8_t* __restrict__ diverged, int64_t* __restrict__ steps_out,
               int64_t* __restrict__ mvms_out) {
    extern __shared__ double sm[];
    const int64_t prob = blockIdx.x / chunks;
    const int chunk = blockIdx.x % chunks;
    if (prob >= P) return;
    const int lane = threadIdx.x;
    const int S = 2 * N + 1;
    double* G = sm;                 // N*N
    double* g = G + N * N;          // N
    double* b = g + N;              // N
    double* X = b + N;              // S*32
    double* E = X + S * kLanes;     // S*32
    double* C = E + S * kLanes;     // S*32
    double* V = C + S * kLanes;     // N*32

    const double* Gp = Gall + prob * (int64_t)N * N;
    for (int i = lane; i < N * N; i += kLanes) G[i] = Gp[i];
    for (int i = lane; i < N; i += kLanes) {
        g[i] = gall[prob * N + i];
        b[i] = ball[prob * N + i];
    }
    __syncwarp();

    const int r = chunk * kLanes + lane;  // anneal index within the problem
    if (r >= B) return;
    const double eps = eps_p ? eps_p[prob] : s.eps;

    // initial state: caller-supplied x0 or the replayed default_rng stream
    if (x0all) {
        const double* x0 = x0all + (prob * B + r) * (int64_t)S;
        for (int i = 0; i < S; ++i) X[i * kLanes + lane] = x0[i];
    } else if (s.rng == IL_RNG_PHILOX) {
        for (int blk = 0; 4 * blk < S; ++blk) {
            float v[4];
            philox_x0_block(base_seed[prob], (uint32_t)r, (uint32_t)blk, (float)s.x0_lo,
                            (float)s.x0_range, v);
            for (int q = 0; q < 4 && 4 * blk + q < S; ++q) X[(4 * blk + q) * kLanes + lane] = v[q];
        }
    } else {
        Pcg64 rng;
        rng.seed_from(derive_seed2(base_seed[prob], (uint64_t)r));
        for (int i = 0; i < S; ++i) X[i * kLanes + lane] = rng.uniform(s.x0_lo, s.x0_range);
    }
    for (int i = 0; i < S; ++i) {
        E[i * kLanes + lane] = 1.0;
        C[i * kLanes + lane] = 0.0;
    }

    const double pm1 = s.p - 1.0;
    const double nzeta = -s.zeta;
    int64_t n_mvm = 0;
    int halted_at = -1;
    for (int t = 0; t < s.n_steps; ++t) {
        if (t % s.f_mvm == 0) {
            const double xa = X[2 * N * kLanes + lane];
            double bdot = 0.0;
            for (int i = 0; i < N; ++i) {
                double vi = dadd(X[i * kLanes + lane], X[(N + i) * kLanes + lane]);
                V[i * kLanes + lane] = vi;
                bdot = dadd(bdot, dmul(b[i], vi));
            }
            // four output rows at a time: each row's sum still runs over j in
            // order (bit-identical), the four dependent chains interleave
            int i = 0;
            for (; i + 4 <= N; i += 4) {
                double acc[4] = {0.0, 0.0, 0.0, 0.0};
                for (int j = 0; j < N; ++j) {
                    const double vj = V[j * kLanes + lane];
#pragma unroll
                    for (int q = 0; q < 4; ++q) acc[q] = dadd(acc[q], dmul(G[(i + q) * N + j], vj));
                }
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const double bx = dmul(b[i + q], xa);
                    C[(i + q) * kLanes + lane] =
                        dadd(dsub(acc[q], dmul(g[i + q], X[(i + q) * kLanes + lane])), bx);
                    C[(N + i + q) * kLanes + lane] =
                        dadd(dsub(acc[q], dmul(g[i + q], X[(N + i + q) * kLanes + lane])), bx);
                }
            }
            for (; i < N; ++i) {
                double acc = 0.0;
                const double* Gi = G + i * N;
                for (int j = 0; j < N; ++j) acc = dadd(acc, dmul(Gi[j], V[j * kLanes + lane]));
                const double bx = dmul(b[i], xa);
                C[i * kLanes + lane] = dadd(dsub(acc, dmul(g[i], X[i * kLanes + lane])), bx);
                C[(N + i) * kLanes + lane] =
                    dadd(dsub(acc, dmul(g[i], X[(N + i) * kLanes + lane])), bx);
            }
            C[2 * N * kLanes + lane] = bdot;
            ++n_mvm;
        }
        bool bad = false;
#pragma unroll 4
        for (int i = 0; i < S; ++i) {
            double xi = X[i * kLanes + lane];
            double ei = E[i * kLanes + lane];
            const double ci = C[i * kLanes + lane];
            const double x2 = dmul(xi, xi);
            const double dxi = dsub(dsub(dmul(pm1, xi), dmul(x2, xi)), dmul(dmul(eps, ei), ci));
            const double dei = dmul(dmul(nzeta, dsub(x2, s.a)), ei);
            xi = dadd(xi, dmul(s.dt, dxi));
            ei = dadd(ei, dmul(s.dt, dei));
            if (ei < s.e_floor) ei = s.e_floor;
            X[i * kLanes + lane] = xi;
            E[i * kLanes + lane] = ei;
            if (fabs(xi) > s.thr || !isfinite(xi) || !isfinite(ei)) bad = true;
        }
        if (bad) {
            halted_at = t;
            break;
        }
    }
    const int64_t row = prob * B + r;
    int8_t* sp = spins + row * S;
    for (int i = 0; i < S; ++i) sp[i] = (X[i * kLanes + lane] >= 0.0) ? 1 : -1;
    if (diverged) diverged[row] = halted_at >= 0 ? 1 : 0;
    if (steps_out) steps_out[row] = halted_at >= 0 ? (int64_t)halted_at + 1 : (int64_t)s.n_steps;
    if (mvms_out) mvms_out[row] = n_mvm;
}

// Multi-warp form of k_anneal_exact: W warps share one chunk of 32 anneals
// (lane = anneal in every warp).  Warp w owns coupling rows and spins in
// contiguous blocks; each row's sum still runs over j in order and each spin
// is updated by exactly the same operations, so the result is bit-identical
// to k_anneal_exact.  A lane that halts stops updating but keeps taking part
// in the CTA barriers; the loop ends when no anneal of the chunk is active.
// Cuts the latency of one problem ~W-fold (the drop-in plugin call) and runs
// W warps per CTA's shared memory in the batched FP64-exact mode.
template <int W>
__global__ void __launch_bounds__(W * kLanes)
k_anneal_exact_mw(const double* __restrict__ Gall, const double* __restrict__ gall,
                  const double* __restrict__ ball, const double* __restrict__ x0all,
                  const uint64_t* __restrict__ base_seed, const double* __restrict__ eps_p,
                  int64_t P, int N, int B, int chunks, AnnealScalars s,
                  int8_t* __restrict__ spins, uint8_t* __restrict__ diverged,
                  int64_t* __restrict__ steps_out, int64_t* __restrict__ mvms_out) {
    extern __shared__ double sm[];
    __shared__ int bad_s[W][kLanes];
    const int64_t prob = blockIdx.x / chunks;
    const int chunk = blockIdx.x % chunks;
    if (prob >= P) return;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int S = 2 * N + 1;
    double* G = sm;
    double* g = G + N * N;
    double* b = g + N;
    double* X = b + N;
    double* E = X + S * kLanes;
    double* C = E + S * kLanes;
    double* V = C + S * kLanes;
    const double* Gp = Gall + prob * (int64_t)N * N;
    for (int i = threadIdx.x; i < N * N; i += W * kLanes) G[i] = Gp[i];
    for (int i = threadIdx.x; i < N; i += W * kLanes) {
        g[i] = gall[prob * N + i];
        b[i] = ball[prob * N + i];
    }
    const int r = chunk * kLanes + lane;
    const bool real = r < B;
    const double eps = eps_p ? eps_p[prob] : s.eps;
    // rows [r0, r1) of the coupling product, spins [s0, s1) of the update
    const int rows = (N + W - 1) / W, r0 = min(N, w * rows), r1 = min(N, r0 + rows);
    const int spn = (S + W - 1) / W, s0 = min(S, w * spn), s1 = min(S, s0 + spn);
    if (real) {
        if (x0all) {
            const double* x0 = x0all + (prob * B + r) * (int64_t)S;
            for (int i = s0; i < s1; ++i) X[i * kLanes + lane] = x0[i];
        } else if (s.rng == IL_RNG_PHILOX) {  // counter-based: each warp its own spins
            for (int blk = s0 / 4; 4 * blk < s1; ++blk) {
                float v[4];
                philox_x0_block(base_seed[prob], (uint32_t)r, (uint32_t)blk, (float)s.x0_lo,
                                (float)s.x0_range, v);
                for (int q = 0; q < 4; ++q)
                    if (4 * blk + q >= s0 && 4 * blk + q < s1) X[(4 * blk + q) * kLanes + lane] = v[q];
            }
        } else if (w == 0) {  // one stream per anneal, drawn in order
            Pcg64 rng;
            rng.seed_from(derive_seed2(base_seed[prob], (uint64_t)r));
            for (int i = 0; i < S; ++i) X[i * kLanes + lane] = rng.uniform(s.x0_lo, s.x0_range);
        }
    }
    for (int i = s0; i < s1; ++i) {
        E[i * kLanes + lane] = 1.0;
        C[i * kLanes + lane] = 0.0;
    }
    __syncthreads();
    const double pm1 = s.p - 1.0;
    const double nzeta = -s.zeta;
    int64_t n_mvm = 0;
    int halted_at = -1;
    bool active = real;
    for (int t = 0; t < s.n_steps; ++t) {
        if (!__syncthreads_or(active)) break;
        if (t % s.f_mvm == 0) {
            const double xa = X[2 * N * kLanes + lane];
            if (active) {
                for (int i = r0; i < r1; ++i)
                    V[i * kLanes + lane] = dadd(X[i * kLanes + lane], X[(N + i) * kLanes + lane]);
            }
            __syncthreads();
            if (active) {
                if (w == 0) {  // b.v, summed over all i in order
                    double bdot = 0.0;
                    for (int i = 0; i < N; ++i) bdot = dadd(bdot, dmul(b[i], V[i * kLanes + lane]));
                    C[2 * N * kLanes + lane] = bdot;
                }
                int i = r0;
                for (; i + 4 <= r1; i += 4) {
                    double acc[4] = {0.0, 0.0, 0.0, 0.0};
                    for (int j = 0; j < N; ++j) {
                        const double vj = V[j * kLanes + lane];
#pragma unroll
                        for (int q = 0; q < 4; ++q) acc[q] = dadd(acc[q], dmul(G[(i + q) * N + j], vj));
                    }
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        const double bx = dmul(b[i + q], xa);
                        C[(i + q) * kLanes + lane] =
                            dadd(dsub(acc[q], dmul(g[i + q], X[(i + q) * kLanes + lane])), bx);
                        C[(N + i + q) * kLanes + lane] =
                            dadd(dsub(acc[q], dmul(g[i + q], X[(N + i + q) * kLanes + lane])), bx);
                    }
                }
                for (; i < r1; ++i) {
                    double acc = 0.0;
                    for (int j = 0; j < N; ++j) acc = dadd(acc, dmul(G[i * N + j], V[j * kLanes + lane]));
                    const double bx = dmul(b[i], xa);
                    C[i * kLanes + lane] = dadd(dsub(acc, dmul(g[i], X[i * kLanes + lane])), bx);
                    C[(N + i) * kLanes + lane] =
                        dadd(dsub(acc, dmul(g[i], X[(N + i) * kLanes + lane])), bx);
                }
                ++n_mvm;
            }
            __syncthreads();
        }
        bool bad = false;
        if (active) {
#pragma unroll 4
            for (int i = s0; i < s1; ++i) {
                double xi = X[i * kLanes + lane];
                double ei = E[i * kLanes + lane];
                const double ci = C[i * kLanes + lane];
                const double x2 = dmul(xi, xi);
                const double dxi = dsub(dsub(dmul(pm1, xi), dmul(x2, xi)), dmul(dmul(eps, ei), ci));
                const double dei = dmul(dmul(nzeta, dsub(x2, s.a)), ei);
                xi = dadd(xi, dmul(s.dt, dxi));
                ei = dadd(ei, dmul(s.dt, dei));
                if (ei < s.e_floor) ei = s.e_floor;
                X[i * kLanes + lane] = xi;
                E[i * kLanes + lane] = ei;
                if (fabs(xi) > s.thr || !isfinite(xi) || !isfinite(ei)) bad = true;
            }
        }
        bad_s[w][lane] = bad;
        __syncthreads();
        bool any = false;
#pragma unroll
        for (int q = 0; q < W; ++q) any = any || bad_s[q][lane];
        if (active && any) {
            halted_at = t;
            active = false;
        }
        __syncthreads();  // bad_s is rewritten next step
    }
    if (!real) return;
    const int64_t row = prob * B + r;
    int8_t* sp = spins + row * S;
    for (int i = s0; i < s1; ++i) sp[i] = (X[i * kLanes + lane] >= 0.0) ? 1 : -1;
    if (w == 0) {
        if (diverged) diverged[row] = halted_at >= 0 ? 1 : 0;
        if (steps_out) steps_out[row] = halted_at >= 0 ? (int64_t)halted_at + 1 : (int64_t)s.n_steps;
        if (mvms_out) mvms_out[row] = n_mvm;
    }
}

}  // namespace

size_t exact_smem_bytes(int N) {
    const int S = 2 * N + 1;
    return sizeof(double) * ((size_t)N * N + 2 * N + 3 * (size_t)S * kLanes + (size_t)N * kLanes);
}

int launch_anneal_exact(const double* G, const double* g, const double* b, const double* x0,
                        const uint64_t* base_seed, const double* eps_p, int64_t P, int N, int B,
                        const AnnealScalars& s, int8_t* spins, uint8_t* diverged,
                        int64_t* steps, int64_t* mvms, cudaStream_t st) {
    if (P == 0 || B == 0) return IL_OK;
    const size_t smem = exact_smem_bytes(N);
    IL_REQUIRE(smem <= 220 * 1024, "n_dim=%d too large for the exact kernel", N);
    IL_CHECK_CUDA(cudaFuncSetAttribute(k_anneal_exact, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)smem));
    const int chunks = (B + kLanes - 1) / kLanes;
    const int64_t blocks = P * chunks;
    IL_REQUIRE(blocks < (1ll << 31), "too many problems in one launch");
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (N >= 8 && IL_EXACT_WARPS > 1) {
        // latency mode (a few problems, e.g. the per-RE plugin call): 8 warps
        // per chunk; throughput mode: 4 warps share a chunk's shared memory
        if (blocks < 2 * (int64_t)sms) {
            IL_CHECK_CUDA(cudaFuncSetAttribute(k_anneal_exact_mw<8>,
                                               cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
            IL_LAUNCH(kProfAnneal, st, k_anneal_exact_mw<8><<<(unsigned)blocks, 8 * kLanes, smem, st>>>(G, g, b, x0, base_seed, eps_p, P, N, B, chunks, s, spins, diverged, steps, mvms););
        } else {
            constexpr int W = IL_EXACT_WARPS;
            IL_CHECK_CUDA(cudaFuncSetAttribute(k_anneal_exact_mw<W>,
                                               cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
            IL_LAUNCH(kProfAnneal, st, k_anneal_exact_mw<W><<<(unsigned)blocks, W * kLanes, smem, st>>>(G, g, b, x0, base_seed, eps_p, P, N, B, chunks, s, spins, diverged, steps, mvms););
        }
    } else {
        IL_LAUNCH(kProfAnneal, st, k_anneal_exact<<<(unsigned)blocks, kLanes, smem, st>>>(G, g, b, x0, base_seed, eps_p, P, N, B,
                                                               chunks, s, spins, diverged, steps, mvms););
    }
    IL_CHECK_CUDA(cudaGetLastError());
    return IL_OK;
}

}  // namespace il
