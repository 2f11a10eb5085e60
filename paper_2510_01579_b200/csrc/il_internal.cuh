// Internal launch interfaces shared by the .cu translation units.
#pragma once
#include <cstdlib>
#include "il_common.cuh"

namespace il {

// Scalars of one anneal batch (CacParams after eps resolution).
struct AnnealScalars {
    double p, a, zeta, eps, dt, e_floor, thr;
    double x0_lo, x0_range;  // uniform(lo, lo + range): lo = -amp, range = amp - (-amp)
    int f_mvm, n_steps;
    int rng = 0;  // il_rng
};

// ---- anneal kernels --------------------------------------------------------
// Exact FP64 (bit-identical to _kernel.pyx).  x0 == nullptr => generate from
// base_seed[p] (anneal r seeded with derive_seed(base_seed[p], r)).
// eps_p == nullptr => s.eps for every problem.
int launch_anneal_exact(const double* G, const double* g, const double* b, const double* x0,
                        const uint64_t* base_seed, const double* eps_p, int64_t P, int N, int B,
                        const AnnealScalars& s, int8_t* spins, uint8_t* diverged,
                        int64_t* steps, int64_t* mvms, cudaStream_t st);

// FP32 state + tensor-core coupling product.  Requires 1 <= N <= 64 (N not
// a multiple of 8 runs with inert padding spins), B % 16 == 0.  Divergence
// is a sticky flag (spins of diverged anneals are not frozen: they never
// enter selection).  steps / mvms (optional, [P][count_rows]): per-anneal
// step and refresh counts as the reference kernel reports them.
// Energies: the FP64 energy of every anneal; or, with screen_rows > 0, only of
// the anneals among the first screen_rows rows of each problem that can be the
// FP64 argmin of those rows (+inf for the others): an FP32 tensor-core
// screen bounds every energy to within 2^-13 (sum|G| + sum|b|) and only the
// distinct configurations within twice that of the minimum are evaluated in
// FP64.  The argmin (ties -> lowest row) is the same.
int launch_anneal_fast(const double* G, const double* g, const double* b,
                       const uint64_t* base_seed, const double* eps_p, int64_t P, int N, int B,
                       const AnnealScalars& s, int precision, int8_t* spins, uint8_t* diverged,
                       double* energies, cudaStream_t st, int screen_rows = 0,
                       int64_t* steps = nullptr, int64_t* mvms = nullptr, int count_rows = 0,
                       const double* gstats = nullptr);
bool fast_anneal_supported(int N, int B, const AnnealScalars& s);
// launch_anneal_fast hands the shape to the tcgen05 kernel (opt-in)
bool fast_anneal_uses_umma(int N, int B);
// spins per half of the register layout the FP32 kernel runs N on (>= N; 0: none)
int fast_anneal_layout(int N);
// The same anneal with the coupling product on tcgen05 (anneal_umma.cu);
// launch_anneal_fast dispatches to it when enabled and supported.
bool umma_anneal_supported(int N, int B);
int launch_anneal_umma(const double* G, const double* g, const double* b,
                       const uint64_t* base_seed, const double* eps_p, int64_t P, int N, int B,
                       const void* fast_scalars, bool split, bool same_qr, int8_t* spins,
                       uint8_t* diverged, double* energies, bool screened, cudaStream_t st);
// anneal rows per problem the fast kernel runs for B requested anneals
// Anneal rows per problem in the fast kernel: 8 (two problems per warp) for
// n_anneals <= 8, else tiles of 16; the extra rows are seeded by their own
// index and never selected.
// ISINGLINK_PACK=0 (read per call) keeps n_anneals <= 8 in padded 16-row
// tiles: the parity test compares both layouts bit for bit.
inline int fast_rows(int B) {
    const char* e = getenv("ISINGLINK_PACK");
    const bool pack = !(e && *e == '0');
    return (B <= 8 && pack) ? 8 : (B + 15) / 16 * 16;
}

// ---- front-end / reduction kernels -----------------------------------------
// Ising outputs of the front-end kernels (any pointer may be null).
struct IsingOut {
    double *G, *g, *b, *offset, *eps_scale, *eps_out;
    double eps_gain, fixed_eps;
    // optional [P][2]: max |G| and sum |G| + sum |b| (k_front_rows only), read
    // by the fast anneal instead of scanning G
    double* gstats = nullptr;
};
// Register-resident front-end for n_t <= 16 (front_rows.cu).
bool front_rows_supported(int n_r, int n_t);
int launch_front_rows(bool do_mmse, bool do_ising, const double* H, const double* y,
                      const double* s2, int64_t P, int n_r, int n_t, const Alphabet& al,
                      uint8_t* x_idx, double* energy, int8_t* status, const IsingOut& o,
                      cudaStream_t st);
int launch_mmse(const double* H, const double* y, const double* noise_var, int64_t P, int n_r,
                int n_t, const Alphabet& al, uint8_t* x_idx, double* energy, int8_t* status,
                cudaStream_t st);
// Ising around a level-index guess; eps_out[p] = eps_gain * eps_scale (or
// fixed_eps if > 0); guess_energy (optional) = ||y - H x_guess||^2.
int launch_build_ising(const double* H, const double* y, const uint8_t* guess_idx, int64_t P,
                       int n_r, int n_t, const Alphabet& al, double* G, double* g_diag,
                       double* b, double* offset, double* eps_scale, double* eps_out,
                       double eps_gain, double fixed_eps, cudaStream_t st, double* gstats = nullptr);
// VPP front-end: W = H^H (H H^H)^-1 [n_ant x n_u], y_t = W u, H_p = -tau/2 W,
// base energy ||y_t||^2.  status[p] = -1 on Cholesky breakdown.
int launch_zf_vpp_front(const double* H, const double* u, int64_t P, int n_u, int n_ant,
                        double tau, double* W, double* y_t, double* H_p, double* base_energy,
                        int8_t* status, cudaStream_t st);

// ---- selection / decode -----------------------------------------------------
// For each problem: energies of the B anneals (FP64), argmin over survivors
// (ties -> lowest index), fallback test best+offset > guess_energy, decode
// clamp(k_g + s_aux*(s_A+s_B)/2), residual of the decoded vector and the
// strict improvement test (solver.py:256-279, detector.py:48-54).
// x_idx_io holds the guess on entry and the result on exit.
int launch_select_decode(const double* H, const double* y, const double* G, const double* b,
                         const double* offset, const int8_t* spins, const uint8_t* diverged,
                         const double* energies, int64_t P, int n_r, int n_t, int B, int Bs,
                         const Alphabet& al,
                         uint8_t* x_idx_io, double* energy_io, int8_t* source,
                         int32_t* anneal_index, int32_t* diverged_count, cudaStream_t st);

int launch_mmse_ising(const double* H, const double* y, const double* noise_var, int64_t P,
                      int n_r, int n_t, const Alphabet& al, uint8_t* x_idx, double* energy,
                      int8_t* status, double* G, double* g_diag, double* b, double* offset,
                      double* eps_out, double eps_gain, double fixed_eps, cudaStream_t st,
                      double* gstats = nullptr);
// MMGaP-E (multi.cu)
int launch_mmse_sic(const double* H, const double* y, const double* noise_var, int64_t P, int n_r,
                    int n_t, const Alphabet& al, uint8_t* x_idx, double* energy, int8_t* status,
                    cudaStream_t st);
int launch_multi_init(const uint8_t* bx, const double* be, const int8_t* bst,
                      const int32_t* codes, int n_chains, int64_t P, int nx, uint8_t* x,
                      double* e, int8_t* src, int32_t* aidx, cudaStream_t st);
int launch_multi_stage(const int32_t* stage_ai, int64_t P, int32_t* widx, cudaStream_t st);
int launch_multi_combine(const uint8_t* gx, const double* ge, const int32_t* widx, int64_t P,
                         int nx, uint8_t* x, double* e, int8_t* src, int32_t* aidx,
                         cudaStream_t st);
int launch_ml_llr(const double* H, const double* y, const double* noise_var, int64_t P, int n_r,
                  int n_t, const Alphabet& al, double* llr, cudaStream_t st);
int launch_ml(const double* H, const double* y, int64_t P, int n_r, int n_t, const Alphabet& al,
              uint8_t* x_idx, double* energy, cudaStream_t st);
int launch_spin_energies(const double* G, const double* b, const int8_t* spins, int64_t P, int B,
                         int N, double* out, cudaStream_t st);
int launch_vpp_post(const double* W, const double* u, const double* y_t, const double* base_energy,
                    const uint8_t* vidx, int64_t P, int n_u, int n_ant, int reach, double tau,
                    double power, double* x, double* v, double* unnorm_power, cudaStream_t st);
int launch_residual(const double* H, const double* y, const double* x, int64_t P, int n_r, int n_t,
                    double* out, cudaStream_t st);
int launch_add_i32(const int32_t* a, int64_t n, int32_t* acc, cudaStream_t st);
int launch_gray_demap(const uint8_t* x_idx, int64_t n_sym, int bits_per_dim, uint8_t* bits,
                      cudaStream_t st);

int launch_base_seeds(const uint64_t* seed, int64_t P, uint64_t k1, uint64_t k2,
                      uint64_t* base_out, cudaStream_t st);

// ---- TMA bulk copy + mbarrier (sm_90+ PTX, used here on sm_100a) -----------
IL_D uint32_t smem_u32(const void* p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}
IL_D void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
IL_D void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}
IL_D void tma_bulk_g2s(void* dst, const void* src, uint32_t bytes,
                                             uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}
IL_D void mbar_wait(uint64_t* bar, uint32_t parity) {
    uint32_t done = 0;
    do {
        asm volatile(
            "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
            " selp.u32 %0, 1, 0, p;\n}\n"
            : "=r"(done)
            : "r"(smem_u32(bar)), "r"(parity)
            : "memory");
    } while (!done);
}

// ---- measurement hooks (prof.cu) -------------------------------------------
enum ProfKind { kProfFront = 0, kProfAnneal = 1, kProfSelect = 2, kProfOther = 3 };
int prof_start(int kind, cudaStream_t st);  // counts the launch; events only when profiling
void prof_stop(int idx, cudaStream_t st);

#define IL_LAUNCH(kind, st, ...)                          \
    do {                                                  \
        const int _pi = ::il::prof_start((kind), (st));   \
        __VA_ARGS__;                                      \
        ::il::prof_stop(_pi, (st));                       \
    } while (0)

// ---- workspace (stream-ordered allocations from the library's pool) --------
// pool_alloc: cudaMallocFromPoolAsync from the library's private per-device
// pool (abi.cu); the memory is released with cudaFreeAsync.
int pool_alloc(void** p, size_t bytes, cudaStream_t st);

struct Workspace {
    cudaStream_t st;
    void* ptrs[32];
    int n = 0;
    explicit Workspace(cudaStream_t s);
    ~Workspace();
    template <class T>
    T* get(size_t count, int* rc) {
        if (*rc != IL_OK) return nullptr;
        if (n >= 32) {
            set_error("workspace: too many buffers");
            *rc = IL_ERR_CUDA;
            return nullptr;
        }
        void* p = nullptr;
        *rc = pool_alloc(&p, count * sizeof(T), st);
        if (*rc != IL_OK) return nullptr;
        ptrs[n++] = p;
        return static_cast<T*>(p);
    }
};

}  // namespace il
