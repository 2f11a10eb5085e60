// Per-problem solve API: the reference's solve_batch / integrate_anneal
// (solver.py:217-279) for P problems whose Ising coefficients are given.
//   il_spin_energies  E(s) for spin vectors (solver.py:171-175)
//   il_solve_batch    anneal -> energies -> best survivor -> fallback test
#include "il_internal.cuh"

namespace il {
namespace {

// FP64 energy of each spin row; one warp per problem, lane = spin row.
__global__ void k_spin_energies(const double* __restrict__ Gg, const double* __restrict__ bg,
                                const int8_t* __restrict__ spins, int64_t P, int B, int N,
                                double* __restrict__ out) {
    extern __shared__ double sm[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t prob = (int64_t)blockIdx.x * (blockDim.x >> 5) + warp;
    if (prob >= P) return;
    const int S = 2 * N + 1;
    double* G = sm + (size_t)warp * (N * N + N);
    double* b = G + N * N;
    for (int i = lane; i < N * N; i += 32) G[i] = Gg[prob * (int64_t)N * N + i];
    for (int i = lane; i < N; i += 32) b[i] = bg[prob * N + i];
    __syncwarp();
    double gsum = 0.0;
    for (int i = 0; i < N; ++i) gsum += G[i * N + i];
    for (int a = lane; a < B; a += 32) {
        const int8_t* s = spins + (prob * B + a) * (int64_t)S;
        double quad = 0.0, lin = 0.0;
        for (int i = 0; i < N; ++i) {
            const double ui = (double)(s[i] + s[N + i]);
            double gu = 0.0;
            for (int j = 0; j < N; ++j) gu += G[i * N + j] * (double)(s[j] + s[N + j]);
            quad += ui * gu;
            lin += b[i] * ui;
        }
        out[prob * B + a] = (quad - 2.0 * gsum) + 2.0 * (double)s[2 * N] * lin;
    }
}

// Coupling field of solver.py:147-168 for P problems: v = x1 + x2, m = G v,
// out = [m - g x1 + b xa, m - g x2 + b xa, b.v].  One warp per problem, lane
// i (+32..) owns row i; the row sum runs over j in order.
__global__ void k_structured_mvm(const double* __restrict__ Gg, const double* __restrict__ gg,
                                 const double* __restrict__ bg, const double* __restrict__ x1g,
                                 const double* __restrict__ x2g, const double* __restrict__ xag,
                                 int64_t P, int N, double* __restrict__ out) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t prob = (int64_t)blockIdx.x * (blockDim.x >> 5) + warp;
    if (prob >= P) return;
    const double* G = Gg + prob * (int64_t)N * N;
    const double* x1 = x1g + prob * N;
    const double* x2 = x2g + prob * N;
    const double* b = bg + prob * N;
    const double* gd = gg + prob * N;
    const double xa = xag[prob];
    double* o = out + prob * (int64_t)(2 * N + 1);
    double bv = 0.0;
    for (int i = lane; i < N; i += 32) {
        double m = 0.0;
        for (int j = 0; j < N; ++j) m = fma(G[(int64_t)i * N + j], x1[j] + x2[j], m);
        o[i] = (m - gd[i] * x1[i]) + b[i] * xa;
        o[N + i] = (m - gd[i] * x2[i]) + b[i] * xa;
        bv = fma(b[i], x1[i] + x2[i], bv);
    }
    bv = warp_sum(bv);
    if (lane == 0) o[2 * N] = bv;
}

// Best non-diverged anneal (strict <, lowest index wins), fallback test,
// and the winner's spins.  One warp per problem.
__global__ void k_select_best(const double* __restrict__ energies, const uint8_t* __restrict__ div,
                              const int8_t* __restrict__ spins, const double* __restrict__ offset,
                              const double* __restrict__ fallback, int64_t P, int B, int Bs, int S,
                              int8_t* __restrict__ best_spins, double* __restrict__ best_energy,
                              int32_t* __restrict__ best_index, int32_t* __restrict__ ndiv_out) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t prob = (int64_t)blockIdx.x * (blockDim.x >> 5) + warp;
    if (prob >= P) return;
    double be = INFINITY;
    int bi = -1, nd = 0;
    for (int a = lane; a < B; a += 32) {
        const bool d = div[prob * Bs + a] != 0;
        nd += d;
        const double e = d ? INFINITY : energies[prob * Bs + a];
        if (e < be) {
            be = e;
            bi = a;
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const double oe = __shfl_xor_sync(0xffffffffu, be, o);
        const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
        if (oe < be || (oe == be && oi >= 0 && (bi < 0 || oi < bi))) {
            be = oe;
            bi = oi;
        }
    }
    nd = __reduce_add_sync(0xffffffffu, nd);
    if (!(be < INFINITY)) bi = -1;
    const bool keep = bi >= 0 && !(be + offset[prob] > fallback[prob]);
    if (lane == 0) {
        if (ndiv_out) ndiv_out[prob] = nd;
        if (best_energy) best_energy[prob] = be;
        if (best_index) best_index[prob] = keep ? bi : -1;
    }
    if (best_spins && bi >= 0) {
        const int8_t* s = spins + (prob * Bs + bi) * (int64_t)S;
        for (int i = lane; i < S; i += 32) best_spins[prob * S + i] = s[i];
    }
}

}  // namespace

int launch_spin_energies(const double* G, const double* b, const int8_t* spins, int64_t P, int B,
                         int N, double* out, cudaStream_t st) {
    if (P == 0 || B == 0) return IL_OK;
    const size_t per_warp = sizeof(double) * ((size_t)N * N + N);
    int wpb = (int)((160 * 1024) / per_warp);
    wpb = wpb < 1 ? 1 : (wpb > 4 ? 4 : wpb);
    const size_t smem = per_warp * wpb;
    IL_REQUIRE(smem <= 227 * 1024, "n_dim too large");
    IL_CHECK_CUDA(cudaFuncSetAttribute(k_spin_energies, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)smem));
    const int blocks = (int)((P + wpb - 1) / wpb);
    IL_LAUNCH(kProfSelect, st,
              k_spin_energies<<<blocks, 32 * wpb, smem, st>>>(G, b, spins, P, B, N, out));
    IL_CHECK_CUDA(cudaGetLastError());
    return IL_OK;
}

}  // namespace il

using namespace il;

extern "C" {

int il_spin_energies(const double* G, const double* g_diag, const double* b, const int8_t* spins,
                     int64_t P, int32_t n_batch, int32_t n_dim, double* energies, void* stream) {
    (void)g_diag;  // tr G is read from G's diagonal, as the reference sums g_diag = diag(G)
    IL_REQUIRE(P >= 0 && n_batch >= 0 && n_dim >= 0, "negative shape");
    return launch_spin_energies(G, b, spins, P, n_batch, n_dim, energies, (cudaStream_t)stream);
}

int il_structured_mvm_batch(const double* G, const double* g_diag, const double* b,
                            const double* x1, const double* x2, const double* xa, int64_t P,
                            int32_t n_dim, double* out, void* stream) {
    IL_REQUIRE(P >= 0 && n_dim >= 1, "invalid shape");
    if (P == 0) return IL_OK;
    cudaStream_t st = (cudaStream_t)stream;
    const int wpb = 4;
    IL_LAUNCH(kProfOther, st, k_structured_mvm<<<(unsigned)((P + wpb - 1) / wpb), 32 * wpb, 0, st>>>(
                                  G, g_diag, b, x1, x2, xa, P, n_dim, out););
    IL_CHECK_CUDA(cudaGetLastError());
    return IL_OK;
}

int il_zf_batch(const double* H, int64_t P, int32_t n_u, int32_t n_ant, double* W, int8_t* status,
                void* stream) {
    IL_REQUIRE(P >= 0 && n_u >= 1 && n_ant >= n_u && n_ant <= 32,
               "zero forcing requires 1 <= n_u <= n_ant <= 32");
    IL_REQUIRE(P == 0 || (H && W && status), "NULL buffer");
    if (P == 0) return IL_OK;
    cudaStream_t st = (cudaStream_t)stream;
    Workspace ws(st);
    int rc = IL_OK;
    // the VPP front end's ZF stage, with the symbol-dependent outputs discarded
    double* u = ws.get<double>((size_t)P * n_u * 2, &rc);
    double* y_t = ws.get<double>((size_t)P * n_ant * 2, &rc);
    double* H_p = ws.get<double>((size_t)P * n_ant * n_u * 2, &rc);
    double* base = ws.get<double>((size_t)P, &rc);
    if (rc) return rc;
    IL_CHECK_CUDA(cudaMemsetAsync(u, 0, sizeof(double) * (size_t)P * n_u * 2, st));
    return launch_zf_vpp_front(H, u, P, n_u, n_ant, 0.0, W, y_t, H_p, base, status, st);
}

int il_solve_batch(const double* G, const double* g_diag, const double* b, const double* offset,
                   const double* fallback_energy, const double* eps, const uint64_t* base_seed,
                   int64_t P, int32_t n_dim, const il_cac_params* prm, int8_t* best_spins,
                   double* best_energy, int32_t* best_index, int32_t* diverged_count,
                   int64_t* steps, int64_t* mvms, void* stream) {
    IL_REQUIRE(prm != nullptr, "params must not be NULL");
    IL_REQUIRE(P >= 0 && n_dim >= 1 && n_dim <= 128, "invalid shape");
    IL_REQUIRE(prm->dt > 0 && prm->f_mvm >= 1 && prm->n_steps >= 1 && prm->n_anneals >= 1,
               "invalid solver parameters");
    if (P == 0) return IL_OK;
    cudaStream_t st = (cudaStream_t)stream;
    const int N = n_dim, S = 2 * N + 1, B = prm->n_anneals;
    AnnealScalars s{};
    s.p = prm->p;
    s.a = prm->a;
    s.zeta = prm->zeta;
    s.dt = prm->dt;
    s.e_floor = prm->e_floor;
    s.thr = prm->diverge_threshold;
    s.x0_lo = -prm->init_amplitude;
    s.x0_range = prm->init_amplitude - (-prm->init_amplitude);
    s.f_mvm = prm->f_mvm;
    s.n_steps = prm->n_steps;
    IL_REQUIRE(prm->rng == IL_RNG_NUMPY || prm->rng == IL_RNG_PHILOX, "unknown rng %d", prm->rng);
    s.rng = prm->rng;
    int rc = IL_OK;
    Workspace ws(st);
    // counters (steps / mvms) are reported by both kernels, so asking for
    // them does not change the arithmetic (the precision alone selects it)
    const bool want_counts = steps != nullptr || mvms != nullptr;
    const bool fast = prm->precision != IL_PREC_FP64_EXACT &&
                      fast_anneal_supported(N, fast_rows(B), s);
    const int Bs = fast ? fast_rows(B) : B;  // padded rows are never selected
    int8_t* spins = ws.get<int8_t>((size_t)P * Bs * S, &rc);
    uint8_t* div = ws.get<uint8_t>((size_t)P * Bs, &rc);
    double* en = ws.get<double>((size_t)P * Bs, &rc);
    if (want_counts && !steps) steps = ws.get<int64_t>((size_t)P * B, &rc);
    if (want_counts && !mvms) mvms = ws.get<int64_t>((size_t)P * B, &rc);
    if (rc) return rc;
    if (fast) {
        rc = launch_anneal_fast(G, g_diag, b, base_seed, eps, P, N, Bs, s, prm->precision, spins,
                                div, en, st, 0, steps, mvms, B);
        if (rc) return rc;
    } else {
        rc = launch_anneal_exact(G, g_diag, b, nullptr, base_seed, eps, P, N, B, s, spins, div, steps,
                                 mvms, st);
        if (rc) return rc;
        rc = launch_spin_energies(G, b, spins, P, B, N, en, st);
        if (rc) return rc;
    }
    const int wpb = 4;
    IL_LAUNCH(kProfSelect, st,
              k_select_best<<<(unsigned)((P + wpb - 1) / wpb), 32 * wpb, 0, st>>>(
                  en, div, spins, offset, fallback_energy, P, B, Bs, S, best_spins, best_energy,
                  best_index, diverged_count));
    IL_CHECK_CUDA(cudaGetLastError());
    return IL_OK;
}

int il_integrate_batch(const double* G, const double* g_diag, const double* b, const double* eps,
                       const uint64_t* seed, int64_t P, int32_t n_dim, const il_cac_params* prm,
                       int8_t* spins, uint8_t* diverged, int64_t* steps, int64_t* mvms,
                       double* energy, void* stream) {
    IL_REQUIRE(prm != nullptr, "params must not be NULL");
    IL_REQUIRE(P >= 0 && n_dim >= 1 && n_dim <= 128, "invalid shape");
    IL_REQUIRE(prm->dt > 0 && prm->f_mvm >= 1 && prm->n_steps >= 1, "invalid solver parameters");
    IL_REQUIRE(P == 0 || (spins && diverged && steps && mvms && seed && eps), "NULL buffer");
    if (P == 0) return IL_OK;
    cudaStream_t st = (cudaStream_t)stream;
    const int N = n_dim, S = 2 * N + 1;
    AnnealScalars s{};
    s.p = prm->p;
    s.a = prm->a;
    s.zeta = prm->zeta;
    s.dt = prm->dt;
    s.e_floor = prm->e_floor;
    s.thr = prm->diverge_threshold;
    s.x0_lo = -prm->init_amplitude;
    s.x0_range = prm->init_amplitude - (-prm->init_amplitude);
    s.f_mvm = prm->f_mvm;
    s.n_steps = prm->n_steps;
    IL_REQUIRE(prm->rng == IL_RNG_NUMPY || prm->rng == IL_RNG_PHILOX, "unknown rng %d", prm->rng);
    s.rng = prm->rng;
    int rc = IL_OK;
    Workspace ws(st);
    double* x0 = ws.get<double>((size_t)P * S, &rc);
    if (rc) return rc;
    // integrate_anneal draws x0 from default_rng(seed) itself (solver.py:227)
    rc = il_initial_states(seed, P, S, prm->init_amplitude, x0, st);
    if (rc) return rc;
    rc = launch_anneal_exact(G, g_diag, b, x0, nullptr, eps, P, N, 1, s, spins, diverged, steps,
                             mvms, st);
    if (rc) return rc;
    return energy ? launch_spin_energies(G, b, spins, P, 1, N, energy, st) : IL_OK;
}

}  // extern "C"
