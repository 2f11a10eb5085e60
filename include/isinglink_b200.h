/*
 * isinglink_b200 — C ABI of the B200-native MMGaP hot path.
 *
 * Drop-in boundary for the reference package `isinglink`
 * (/root/reference/pkg/src/isinglink).  Every entry point below states the
 * reference interface it replaces (file:line).  Conventions:
 *   - plain pointers and sizes only; no torch / numpy types;
 *   - functions named *_host take HOST pointers and are synchronous; all
 *     others take DEVICE pointers and enqueue on `stream` (a cudaStream_t,
 *     NULL = legacy default stream) without synchronising;
 *   - complex arrays are interleaved (re, im) float64, i.e. numpy complex128
 *     / torch.complex128 memory; the detection entries stage H and y with
 *     16-byte asynchronous copies and require them 16-byte aligned (every
 *     CUDA allocation and every complex128 element of one is), else IL_ERR_ARG;
 *   - return 0 (IL_OK) on success, a negative IL_ERR_* code otherwise, with a
 *     human-readable message from il_last_error() (thread-local).  No C++
 *     exception ever crosses the ABI.  Divergence of an anneal is data, not
 *     an error (as in the reference).
 */
#ifndef ISINGLINK_B200_H
#define ISINGLINK_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define IL_ABI_VERSION 2

enum il_status {
    IL_OK = 0,
    IL_ERR_ARG = -1,         /* invalid argument (reference: ValueError/TypeError) */
    IL_ERR_CUDA = -2,        /* CUDA runtime / launch failure */
    IL_ERR_UNSUPPORTED = -3, /* shape/parameter combination not built */
    IL_ERR_NOMEM = -4
};

/* Arithmetic of the anneal loop. */
enum il_precision {
    IL_PREC_FP64_EXACT = 0, /* FP64, reference evaluation order, no FMA contraction:
                               bit-identical to the reference "ext" kernel */
    IL_PREC_FP32 = 1,       /* FP32 state, coupling product on tensor cores as a
                               3-pass f16 hi/lo split (hi*hi + lo*hi + hi*lo, FP32
                               accumulate; FP32-accurate); the throughput mode */
    IL_PREC_TF32 = 2,       /* FP32 state, single-pass f16 coupling product
                               (11-bit significand, like TF32) */
    IL_PREC_MIXED = 3       /* FP32 state; coupling product as IL_PREC_FP32 for the
                               first 16 steps, then 2 passes (hi*hi + hi*lo: G split
                               to FP32 accuracy, the state rounded to f16) */
};

/* Solver configuration — mirrors CacParams (solver.py:87-124). */
typedef struct il_cac_params {
    double p;                 /* gain                                  (1.5)  */
    double a;                 /* target amplitude^2                    (0.5)  */
    double zeta;              /* error-variable rate                   (1.0)  */
    double eps;               /* coupling; <= 0 selects auto scaling   (auto) */
    double dt;                /* Euler step                            (0.02) */
    int32_t f_mvm;            /* coupling refresh period               (2)    */
    int32_t n_steps;          /*                                       (128)  */
    int32_t n_anneals;        /* replicas per problem                  (32)   */
    int32_t precision;        /* il_precision                                 */
    double diverge_threshold; /*                                       (10.0) */
    double e_floor;           /*                                       (1e-6) */
    double init_amplitude;    /*                                       (0.1)  */
    int32_t rng;              /* il_rng: initial-state generator              */
    int32_t reserved;         /* must be 0                                    */
} il_cac_params;

/* Initial-state generator (solver.py:182-187 draws default_rng(derive_seed(
 * seed, r)).uniform(-amp, amp, 2N + 1) per anneal r). */
enum il_rng {
    IL_RNG_NUMPY = 0,  /* those numpy streams, replayed bit for bit (SeedSequence + PCG64) */
    IL_RNG_PHILOX = 1  /* counter-based Philox4x32-10 keyed by the same per-problem seed
                          (csrc/rng_philox.cuh): FP32 states, no stream replay; parity is
                          statistical against the reference */
};

/* Per-problem outcome of a batched detection (DetectionResult.source,
 * linear.py:33-41): "mmse" (the guess) = 0, "anneal" = 1, "mmse_sic" = 2
 * (detect_cim_multi only), -1 = the baseline's Cholesky failed (the
 * reference raises LinAlgError there). */
enum il_source { IL_SRC_GUESS = 0, IL_SRC_ANNEAL = 1, IL_SRC_SIC = 2, IL_SRC_FAILED = -1 };

const char* il_last_error(void);
int il_abi_version(void);

/* Which anneal kernel the batched entries run for n_dim spins per half
 * (N = 2 n_t), n_anneals replicas and these parameters (no GPU work):
 * IL_KERNEL_EXACT (FP64, bit-identical; always for IL_PREC_FP64_EXACT),
 * IL_KERNEL_FAST (FP32 + tensor cores, N a multiple of 8),
 * IL_KERNEL_FAST_PADDED (the same with inert padding spins up to the next
 * built layout), IL_KERNEL_UMMA (tcgen05 coupling product, opt-in), or a
 * negative IL_ERR_* for invalid parameters. */
enum il_anneal_kernel {
    IL_KERNEL_EXACT = 0,
    IL_KERNEL_FAST = 1,
    IL_KERNEL_FAST_PADDED = 2,
    IL_KERNEL_UMMA = 3
};
int il_anneal_kernel(int32_t n_dim, const il_cac_params* prm);

/* ---------------------------------------------------------------------------
 * Kernel plugin: replaces `_kernel.run_anneals` (_kernel.pyx:16-102, contract
 * _kernel_py.py:24-92).  G[n_dim*n_dim], g_diag[n_dim], b[n_dim],
 * x0[n_batch*(2*n_dim+1)] row-major float64.  Outputs: spins int8
 * [n_batch*(2*n_dim+1)] with sign(0)=+1, diverged uint8[n_batch],
 * steps int64[n_batch], mvms int64[n_batch].  Always FP64-exact.
 * ------------------------------------------------------------------------- */
int il_run_anneals(const double* G, const double* g_diag, const double* b,
                   const double* x0, int32_t n_dim, int32_t n_batch, double dt,
                   double p, double a, double zeta, double eps, double e_floor,
                   int32_t f_mvm, int32_t n_steps, double diverge_threshold,
                   int8_t* spins, uint8_t* diverged, int64_t* steps, int64_t* mvms,
                   void* stream);
int il_run_anneals_host(const double* G, const double* g_diag, const double* b,
                        const double* x0, int32_t n_dim, int32_t n_batch, double dt,
                        double p, double a, double zeta, double eps, double e_floor,
                        int32_t f_mvm, int32_t n_steps, double diverge_threshold,
                        int8_t* spins, uint8_t* diverged, int64_t* steps,
                        int64_t* mvms);

/* ---------------------------------------------------------------------------
 * Seeds and initial states.
 *   il_derive_seeds: out[i] = derive_seed(parts[i*n_parts + 0..n_parts))
 *     (solver.py:137-144, numpy SeedSequence), n_parts <= 6.
 *   il_initial_states: x0[i*S + k] = default_rng(seeds[i]).uniform(-amp, amp, S)[k]
 *     (solver.py:182-187, numpy PCG64), bit-exact.
 * ------------------------------------------------------------------------- */
int il_derive_seeds(const uint64_t* parts, int32_t n_parts, int64_t n, uint64_t* out,
                    void* stream);
int il_initial_states(const uint64_t* seeds, int64_t n, int32_t S, double amplitude,
                      double* x0, void* stream);

/* ---------------------------------------------------------------------------
 * Linear front-end + Ising reduction for P independent problems.
 *   il_mmse_batch — detect_mmse (linear.py:55-75): hard MMSE decision as
 *     level indices x_idx[P*n_t*2] (re, im) and residual energy[P].
 *   il_build_ising_batch — build_ising (transform.py:108-140) around the
 *     guess given as level indices of `levels` (qam_order > 0: unit-energy
 *     QAM; qam_order < 0: VPP lattice of reach -qam_order).  Outputs
 *     G[P*N*N], g_diag[P*N], b[P*N], offset[P], eps_scale[P] (N = 2*n_t).
 * H is [P, n_r, n_t] complex128, y [P, n_r], noise_var [P].
 * status[P] (optional, may be NULL): 0 ok, -1 Cholesky breakdown.
 * ------------------------------------------------------------------------- */
int il_mmse_batch(const double* H, const double* y, const double* noise_var,
                  int64_t P, int32_t n_r, int32_t n_t, int32_t qam_order,
                  uint8_t* x_idx, double* energy, int8_t* status, void* stream);
int il_build_ising_batch(const double* H, const double* y, const uint8_t* guess_idx,
                         int64_t P, int32_t n_r, int32_t n_t, int32_t qam_order,
                         double* G, double* g_diag, double* b, double* offset,
                         double* eps_scale, void* stream);

/* ---------------------------------------------------------------------------
 * Solver on given Ising problems (solver.py:217-279).
 *   il_spin_energies — E(s) = u'Gu - 2 tr G + 2 s_aux b'u, u = s_A + s_B
 *     (solver.py:171-175, transform.py:143-152) for spins[P*n_batch*(2N+1)].
 *   il_solve_batch — P x solve_batch: anneal r of problem p starts from
 *     default_rng(derive_seed(base_seed[p], r)).uniform(-amp, amp); returns
 *     the best non-diverged anneal (strict <, lowest index on ties) in
 *     best_spins[P*(2N+1)], best_energy[P], best_index[P] (-1 when every
 *     anneal diverged or best_energy + offset > fallback_energy, i.e. when
 *     the reference returns None), diverged_count[P].  eps[P] is the
 *     resolved coupling.  steps/mvms [P*n_anneals] (optional): the
 *     reference's per-anneal counters (steps before halting, coupling
 *     refreshes), reported in every precision (they do not change it).
 * ------------------------------------------------------------------------- */
int il_spin_energies(const double* G, const double* g_diag, const double* b,
                     const int8_t* spins, int64_t P, int32_t n_batch, int32_t n_dim,
                     double* energies, void* stream);
/* structured_mvm (solver.py:147-168) for P problems: v = x1 + x2,
 * out[P][2N+1] = [G v - g x1 + b xa, G v - g x2 + b xa, b.v] (FP64). */
int il_structured_mvm_batch(const double* G, const double* g_diag, const double* b,
                            const double* x1, const double* x2, const double* xa, int64_t P,
                            int32_t n_dim, double* out, void* stream);
int il_solve_batch(const double* G, const double* g_diag, const double* b,
                   const double* offset, const double* fallback_energy, const double* eps,
                   const uint64_t* base_seed, int64_t P, int32_t n_dim,
                   const il_cac_params* prm, int8_t* best_spins, double* best_energy,
                   int32_t* best_index, int32_t* diverged_count, int64_t* steps,
                   int64_t* mvms, void* stream);

/* P x integrate_anneal (solver.py:217-235): one FP64-exact anneal per
 * problem from default_rng(seed[p]).uniform(-amp, amp), coupling eps[p];
 * spins[P*(2N+1)], diverged[P], steps[P], mvms[P], energy[P] (may be NULL).
 * Drives the Appendix-A integration heatmap (harness/heatmap.py). */
int il_integrate_batch(const double* G, const double* g_diag, const double* b,
                       const double* eps, const uint64_t* seed, int64_t P, int32_t n_dim,
                       const il_cac_params* prm, int8_t* spins, uint8_t* diverged,
                       int64_t* steps, int64_t* mvms, double* energy, void* stream);

/* Exhaustive ML detection (linear.py:109-144), ties to the smallest symbol-
 * index vector (user 0 most significant); refuses > 24-bit search spaces.
 * x_idx[P*n_t*2] level indices, energy[P] residual (may be NULL). */
int il_ml_batch(const double* H, const double* y, int64_t P, int32_t n_r, int32_t n_t,
                int32_t qam_order, uint8_t* x_idx, double* energy, void* stream);

/* Max-log bit LLRs by the same exhaustive search (n_r <= 16, <= 24 bits).
 * No reference counterpart (soft output is a non-goal of the reference,
 * SPEC.md:153; parity unpinned): llr[P * n_t * 2 * bits_per_dim] with bits in
 * the order of il_gray_demap (user, re then im, MSB first) and
 *   llr = (min_{x: bit = 1} ||y - Hx||^2 - min_{x: bit = 0} ||y - Hx||^2) / s2,
 * s2 = noise_var[p] (1 when noise_var is NULL): positive favours bit 0. */
int il_ml_llr_batch(const double* H, const double* y, const double* noise_var, int64_t P,
                    int32_t n_r, int32_t n_t, int32_t qam_order, double* llr, void* stream);

/* ---------------------------------------------------------------------------
 * Batched uplink detection: P x detect_cim (detector.py:57-82) with
 * seed[p] the `seed` argument of detect_cim for problem p.  Outputs:
 *   x_idx[P*n_t*2] level indices (re, im) of x_hard,
 *   energy[P] residual ||y - H x_hard||^2,
 *   source[P] il_source, anneal_index[P] (-1 unless source == anneal),
 *   diverged_count[P].
 * Any output pointer except x_idx may be NULL.
 * ------------------------------------------------------------------------- */
int il_detect_cim_batch(const double* H, const double* y, const double* noise_var,
                        int64_t P, int32_t n_r, int32_t n_t, int32_t qam_order,
                        const uint64_t* seed, const il_cac_params* prm, uint8_t* x_idx,
                        double* energy, int8_t* source, int32_t* anneal_index,
                        int32_t* diverged_count, void* stream);

/* ---------------------------------------------------------------------------
 * MMGaP-E (detector.py:85-134, linear.py:78-106).
 *   il_mmse_sic_batch — P x detect_mmse_sic: x_idx[P*n_t*2] level indices,
 *     energy[P] residual, status[P] (0 ok, -1 Cholesky failure).
 *   il_detect_cim_multi_batch — P x detect_cim_multi(inst, params, n_stages,
 *     seed[p], chains): chains[n_chains] are chain codes in order
 *     (0 = "mmse", 1 = "mmse_sic"; the reference default is {0, 1});
 *     chain c, stage s anneals with derive_seed(seed[p], c, s).  Outputs as
 *     il_detect_cim_batch with source in {0 mmse, 1 anneal, 2 mmse_sic};
 *     diverged_count[P] sums every chain and stage.
 * ------------------------------------------------------------------------- */
/* ||y - H x||^2 per problem (linear.py:44-47) for complex128 x[P*n_t]; the
 * same arithmetic as every energy the detectors compute. */
int il_residual_batch(const double* H, const double* y, const double* x, int64_t P,
                      int32_t n_r, int32_t n_t, double* energy, void* stream);
int il_mmse_sic_batch(const double* H, const double* y, const double* noise_var, int64_t P,
                      int32_t n_r, int32_t n_t, int32_t qam_order, uint8_t* x_idx,
                      double* energy, int8_t* status, void* stream);
int il_detect_cim_multi_batch(const double* H, const double* y, const double* noise_var,
                              int64_t P, int32_t n_r, int32_t n_t, int32_t qam_order,
                              const uint64_t* seed, const il_cac_params* prm,
                              int32_t n_stages, const int32_t* chains, int32_t n_chains,
                              uint8_t* x_idx, double* energy, int8_t* source,
                              int32_t* anneal_index, int32_t* diverged_count, void* stream);

/* ---------------------------------------------------------------------------
 * Host-buffer form of il_detect_cim_batch: every pointer is HOST memory (the
 * numpy-in / numpy-out shape of the reference's detect_cim over a slot).
 * The slot is streamed through the device in n_chunks pieces (<= 0: auto)
 * with the H2D copy, the detection and the D2H copy of consecutive chunks
 * overlapped on separate streams; returns when the outputs are in host
 * memory.  Pinned (page-locked) host buffers are needed for the overlap.
 * ------------------------------------------------------------------------- */
int il_detect_cim_host(const double* H, const double* y, const double* noise_var,
                       int64_t P, int32_t n_r, int32_t n_t, int32_t qam_order,
                       const uint64_t* seed, const il_cac_params* prm, uint8_t* x_idx,
                       double* energy, int8_t* source, int32_t* anneal_index,
                       int32_t* diverged_count, int32_t n_chunks);

/* Streaming form of il_detect_cim_host: enqueues the same pipeline and
 * returns at once with *ticket; il_pipeline_wait(ticket) returns when the
 * outputs are in host memory (inputs must stay valid until then).  Slots
 * submitted back to back share the device streams, so the copies and the
 * first chunks of slot s+1 overlap the tail of slot s.  *ticket is NULL
 * (nothing to wait for) when P == 0. */
int il_detect_cim_host_submit(const double* H, const double* y, const double* noise_var,
                              int64_t P, int32_t n_r, int32_t n_t, int32_t qam_order,
                              const uint64_t* seed, const il_cac_params* prm, uint8_t* x_idx,
                              double* energy, int8_t* source, int32_t* anneal_index,
                              int32_t* diverged_count, int32_t n_chunks, void** ticket);
int il_pipeline_wait(void* ticket);

/* il_detect_cim_host_submit plus the spin-to-bit demapper in the same
 * pipeline: bits[P * n_t * 2 * log2(sqrt(qam_order))] receives the Gray bits
 * of the decided symbols (il_gray_demap's layout, computed on the device per
 * chunk), so the uplink receiver's output leaves the GPU as bits.  Every
 * output pointer may be NULL (not copied back); x_idx NULL keeps the level
 * indices on the device. */
int il_detect_cim_bits_host_submit(const double* H, const double* y, const double* noise_var,
                                   int64_t P, int32_t n_r, int32_t n_t, int32_t qam_order,
                                   const uint64_t* seed, const il_cac_params* prm,
                                   uint8_t* bits, uint8_t* x_idx, double* energy,
                                   int8_t* source, int32_t* anneal_index,
                                   int32_t* diverged_count, int32_t n_chunks, void** ticket);

/* Host-buffer form of il_precode_vpp_batch (every pointer HOST memory),
 * streamed through the device in n_chunks pieces (<= 0: auto) like
 * il_detect_cim_host. */
int il_precode_vpp_host(const double* H, const double* u, int64_t P, int32_t n_u,
                        int32_t n_ant, double power, double tau, int32_t n_stages,
                        const uint64_t* seed, const il_cac_params* prm, double* x, double* v,
                        double* unnorm_power, int32_t* diverged_count, int32_t n_chunks);

/* ---------------------------------------------------------------------------
 * Batched downlink vector-perturbation precoding: P x precode_vpp
 * (precoder.py:93-146).  H [P, n_u, n_ant] complex128 (n_u <= n_ant),
 * u [P, n_u] complex128 symbols, power P_tot > 0, tau, 0 <= n_stages <= 15,
 * seed[p].  Outputs x[P*n_ant] complex128 transmit vector, v[P*n_u]
 * complex128 perturbation (even Gaussian integers), unnorm_power[P],
 * diverged_count[P] (may be NULL).
 * ------------------------------------------------------------------------- */
/* Zero forcing (precoder.py:54-60) for P channels: W[P][n_ant][n_u] =
 * H^H (H H^H)^-1 by Cholesky; status[p] = -1 where the Cholesky broke down
 * (the reference raises LinAlgError). */
int il_zf_batch(const double* H, int64_t P, int32_t n_u, int32_t n_ant, double* W,
                int8_t* status, void* stream);
int il_precode_vpp_batch(const double* H, const double* u, int64_t P, int32_t n_u,
                         int32_t n_ant, double power, double tau, int32_t n_stages,
                         const uint64_t* seed, const il_cac_params* prm, double* x,
                         double* v, double* unnorm_power, int32_t* diverged_count,
                         void* stream);

/* ---------------------------------------------------------------------------
 * Spin-to-bit demapper (channel.py:160-180 Gray labels).  For n_sym symbols
 * with level indices x_idx[n_sym*2] (re, im) and bits_per_dim = log2(m):
 * bits[n_sym * 2 * bits_per_dim] uint8 in {0,1}, ordered (re MSB..LSB,
 * im MSB..LSB) per symbol.
 * ------------------------------------------------------------------------- */
int il_gray_demap(const uint8_t* x_idx, int64_t n_sym, int32_t bits_per_dim,
                  uint8_t* bits, void* stream);

/* ---------------------------------------------------------------------------
 * Measurement hooks (no reference counterpart; used by bench.py).
 *   il_kernel_launches: cumulative number of kernels this library launched.
 *   il_profile_begin/end: while enabled, every launch is bracketed by CUDA
 *     events on its stream; il_profile_end synchronises and returns summed
 *     milliseconds and launch counts per kind (0 front-end/reduction,
 *     1 anneal, 2 select/decode, 3 other), n_kinds <= 4.
 *   il_probe_fp32_peak: dense FFMA throughput (TFLOP/s) of the current GPU.
 * ------------------------------------------------------------------------- */
long long il_kernel_launches(void);
void il_profile_begin(void);
int il_profile_end(double* ms_by_kind, long long* launches_by_kind, int n_kinds);
int il_probe_fp32_peak(int reps, double* tflops);

#ifdef __cplusplus
}
#endif

#endif /* ISINGLINK_B200_H */
