// extern "C" entry points (include/isinglink_b200.h) and the batched
// pipelines that chain the kernels.  No C++ exception crosses this file's
// boundary; every failure becomes an IL_ERR_* code plus il_last_error().
#include <math.h>
#include <stdarg.h>
#include <stdio.h>
#include <string.h>

#include <algorithm>
#include <cstdlib>
#include <mutex>

#include "il_internal.cuh"
#include "rng_numpy.cuh"

namespace il {

static thread_local char g_err[512] = "";

void set_error(const char* fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof(g_err), fmt, ap);
    va_end(ap);
}

int fail_cuda(cudaError_t e, const char* what) {
    set_error("%s: %s", what, cudaGetErrorString(e));
    return IL_ERR_CUDA;
}

// The library's own stream-ordered memory pool, one per device.  Its
// settings stay private (co-located cudaMallocAsync users of the default
// pool are unaffected):
//   * freed workspace is kept for the next call (release threshold = max);
//   * no stream waits on another stream's free (internal dependencies off):
//     with streamed slots on several streams that serialised them into
//     15-50 ms stalls;
//   * the working set is reserved once (ISINGLINK_POOL_RESERVE_MB, default
//     IL_POOL_RESERVE_MB, at most a quarter of the free memory; 0 = none), so
//     that no call grows the pool: growth blocks the enqueueing thread for
//     10-100 ms.
#ifndef IL_POOL_RESERVE_MB
#define IL_POOL_RESERVE_MB 6144
#endif
static constexpr int kMaxDevices = 64;

int device_pool(cudaMemPool_t* out) {
    static std::once_flag once[kMaxDevices];
    static cudaMemPool_t pools[kMaxDevices];
    static cudaError_t errs[kMaxDevices];
    int dev = 0;
    IL_CHECK_CUDA(cudaGetDevice(&dev));
    IL_REQUIRE(dev >= 0 && dev < kMaxDevices, "device ordinal out of range");
    std::call_once(once[dev], [dev] {
        cudaMemPoolProps props = {};
        props.allocType = cudaMemAllocationTypePinned;
        props.location.type = cudaMemLocationTypeDevice;
        props.location.id = dev;
        cudaError_t e = cudaMemPoolCreate(&pools[dev], &props);
        if (e == cudaSuccess) {
            uint64_t thr = UINT64_MAX;
            int no = 0;
            e = cudaMemPoolSetAttribute(pools[dev], cudaMemPoolAttrReleaseThreshold, &thr);
            if (e == cudaSuccess)
                e = cudaMemPoolSetAttribute(pools[dev], cudaMemPoolReuseAllowInternalDependencies, &no);
        }
        if (e == cudaSuccess) {
            const char* env = getenv("ISINGLINK_POOL_RESERVE_MB");
            const long long mb = env && *env ? atoll(env) : (long long)IL_POOL_RESERVE_MB;
            size_t free_b = 0, total_b = 0;
            if (mb > 0 && cudaMemGetInfo(&free_b, &total_b) == cudaSuccess) {
                const size_t reserve = std::min<size_t>((size_t)mb << 20, free_b / 4);
                cudaStream_t s = nullptr;
                void* p = nullptr;
                if (reserve && cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking) == cudaSuccess) {
                    if (cudaMallocFromPoolAsync(&p, reserve, pools[dev], s) == cudaSuccess)
                        cudaFreeAsync(p, s);
                    cudaStreamSynchronize(s);
                    cudaStreamDestroy(s);
                }
                cudaGetLastError();  // a failed reserve only costs the growth later
            }
        }
        errs[dev] = e;
    });
    if (errs[dev] != cudaSuccess) return fail_cuda(errs[dev], "cudaMemPoolCreate");
    *out = pools[dev];
    return IL_OK;
}

int pool_alloc(void** p, size_t bytes, cudaStream_t st) {
    cudaMemPool_t pool;
    const int rc = device_pool(&pool);
    if (rc) return rc;
    const cudaError_t e = cudaMallocFromPoolAsync(p, bytes ? bytes : 1, pool, st);
    return e == cudaSuccess ? IL_OK : fail_cuda(e, "cudaMallocFromPoolAsync");
}

Workspace::Workspace(cudaStream_t s) : st(s) {}

Workspace::~Workspace() {
    for (int i = 0; i < n; ++i) cudaFreeAsync(ptrs[i], st);
}

int make_qam_alphabet(int order, Alphabet* out) {
    int m = 0;
    switch (order) {
        case 4: m = 2; break;
        case 16: m = 4; break;
        case 64: m = 8; break;
        case 256: m = 16; break;
        default:
            set_error("unsupported QAM order %d; expected one of (4, 16, 64, 256)", order);
            return IL_ERR_ARG;
    }
    // channel.py:88-108: odd integers / sqrt(2 (m^2 - 1) / 3)
    const double norm = sqrt(2.0 * (double)(m * m - 1) / 3.0);
    out->m = m;
    out->spacing = 2.0 / norm;
    for (int k = 0; k < m; ++k) out->levels[k] = (double)(-(m - 1) + 2 * k) / norm;
    for (int k = 0; k + 1 < m; ++k) out->mids[k] = (out->levels[k] + out->levels[k + 1]) / 2.0;
    return IL_OK;
}

int make_lattice_alphabet(int reach, Alphabet* out) {
    // precoder.py:79-90: levels 4 * {-reach..reach}, spacing 4.  reach = 0
    // (n_stages = 0) is the single level 0: no stage runs and v = 0.
    if (reach < 0 || 2 * reach + 1 > 31) {
        set_error("VPP n_stages must be in [0, 15] (the lattice of 2 n_stages + 1 levels per "
                  "dimension is built up to 31 levels), got %d", reach);
        return IL_ERR_ARG;
    }
    out->m = 2 * reach + 1;
    out->spacing = 4.0;
    for (int k = 0; k < out->m; ++k) out->levels[k] = 4.0 * (double)(k - reach);
    for (int k = 0; k + 1 < out->m; ++k) out->mids[k] = (out->levels[k] + out->levels[k + 1]) / 2.0;
    return IL_OK;
}

static int alphabet_for(int qam_order, Alphabet* al) {
    return qam_order > 0 ? make_qam_alphabet(qam_order, al) : make_lattice_alphabet(-qam_order, al);
}

// CacParams.validate (solver.py:109-124)
static int validate(const il_cac_params* p) {
    IL_REQUIRE(p != nullptr, "params must not be NULL");
    IL_REQUIRE(p->dt > 0, "dt must be positive");
    IL_REQUIRE(p->f_mvm >= 1 && p->n_steps >= 1 && p->n_anneals >= 1,
               "f_mvm, n_steps and n_anneals must be >= 1");
    IL_REQUIRE(p->e_floor > 0, "e_floor must be positive");
    IL_REQUIRE(p->init_amplitude > 0, "init_amplitude must be positive");
    const double floor_ = sqrt(fmax(fmax(p->a, p->p - 1.0), 0.0));
    IL_REQUIRE(p->diverge_threshold > floor_,
               "diverge_threshold must exceed sqrt(max(a, p - 1)) = %.3g", floor_);
    IL_REQUIRE(p->precision >= IL_PREC_FP64_EXACT && p->precision <= IL_PREC_MIXED,
               "unknown precision %d", p->precision);
    IL_REQUIRE(p->rng == IL_RNG_NUMPY || p->rng == IL_RNG_PHILOX, "unknown rng %d", p->rng);
    IL_REQUIRE(p->reserved == 0, "il_cac_params.reserved must be 0");
    return IL_OK;
}

static AnnealScalars scalars_of(const il_cac_params* p) {
    AnnealScalars s;
    s.p = p->p;
    s.a = p->a;
    s.zeta = p->zeta;
    s.eps = 0.0;
    s.dt = p->dt;
    s.e_floor = p->e_floor;
    s.thr = p->diverge_threshold;
    s.x0_lo = -p->init_amplitude;
    s.x0_range = p->init_amplitude - (-p->init_amplitude);  // numpy: high - low
    s.f_mvm = p->f_mvm;
    s.n_steps = p->n_steps;
    s.rng = p->rng;
    return s;
}

// One _improve_guess stage for P problems (detector.py:27-54) whose Ising
// problems (G, g, b, offset, eps) are already built around the guess held
// in x_idx/energy: anneal, select, decode, keep-if-strictly-better.
static int anneal_and_select(const double* H, const double* y, int64_t P, int n_r, int n_t,
                             const Alphabet& al, const double* G, const double* g, const double* b,
                             const double* offset, const double* eps, const uint64_t* base,
                             const il_cac_params* prm, uint8_t* x_idx, double* energy,
                             int8_t* source, int32_t* anneal_index, int32_t* diverged_count,
                             cudaStream_t st, const double* gstats = nullptr) {
    Workspace ws(st);  // per stage: released (stream-ordered) when the stage is enqueued
    const int N = 2 * n_t, S = 2 * N + 1, B = prm->n_anneals;
    const AnnealScalars s = scalars_of(prm);
    // the fast kernel runs anneals in tiles of 16: B is padded (anneal r of a
    // problem is seeded by r alone, so the extra rows change nothing) and the
    // selection reads the first B rows of each problem
    const bool fast = prm->precision != IL_PREC_FP64_EXACT &&
                      fast_anneal_supported(N, fast_rows(B), s);
    const int Bs = fast ? fast_rows(B) : B;
    int rc = IL_OK;
    int8_t* spins = ws.get<int8_t>((size_t)P * Bs * S, &rc);
    uint8_t* div = ws.get<uint8_t>((size_t)P * Bs, &rc);
    if (rc) return rc;
    double* energies = nullptr;
    if (fast) {
        // only the argmin matters here: the kernel screens its anneals in FP32
        // and evaluates the near-minimal ones in FP64
        energies = ws.get<double>((size_t)P * Bs, &rc);
        if (rc) return rc;
        rc = launch_anneal_fast(G, g, b, base, eps, P, N, Bs, s, prm->precision, spins, div,
                                energies, st, /*screen_rows=*/B, nullptr, nullptr, 0, gstats);
    } else {
        rc = launch_anneal_exact(G, g, b, nullptr, base, eps, P, N, B, s, spins, div, nullptr,
                                 nullptr, st);
    }
    if (rc) return rc;
    return launch_select_decode(H, y, G, b, offset, spins, div, energies, P, n_r, n_t, B, Bs, al,
                                x_idx, energy, source, anneal_index, diverged_count, st);
}

}  // namespace il

using namespace il;

extern "C" {

const char* il_last_error(void) { return il::g_err; }
int il_abi_version(void) { return IL_ABI_VERSION; }

int il_anneal_kernel(int32_t n_dim, const il_cac_params* prm) {
    int rc = validate(prm);
    if (rc) return rc;
    IL_REQUIRE(n_dim >= 1, "n_dim must be >= 1");
    if (prm->precision == IL_PREC_FP64_EXACT) return IL_KERNEL_EXACT;
    const int B = fast_rows(prm->n_anneals);
    if (!fast_anneal_supported(n_dim, B, scalars_of(prm))) return IL_KERNEL_EXACT;
    if (fast_anneal_uses_umma(n_dim, B)) return IL_KERNEL_UMMA;
    return fast_anneal_layout(n_dim) == n_dim ? IL_KERNEL_FAST : IL_KERNEL_FAST_PADDED;
}

int il_run_anneals(const double* G, const double* g_diag, const double* b, const double* x0,
                   int32_t n_dim, int32_t n_batch, double dt, double p, double a, double zeta,
                   double eps, double e_floor, int32_t f_mvm, int32_t n_steps,
                   double diverge_threshold, int8_t* spins, uint8_t* diverged, int64_t* steps,
                   int64_t* mvms, void* stream) {
    IL_REQUIRE(n_dim >= 0 && n_batch >= 0, "negative shape");
    IL_REQUIRE(f_mvm >= 1, "f_mvm must be >= 1");
    IL_REQUIRE(n_batch == 0 || (x0 && spins && diverged && steps && mvms), "NULL buffer");
    AnnealScalars s{};
    s.p = p;
    s.a = a;
    s.zeta = zeta;
    s.eps = eps;
    s.dt = dt;
    s.e_floor = e_floor;
    s.thr = diverge_threshold;
    s.f_mvm = f_mvm;
    s.n_steps = n_steps < 0 ? 0 : n_steps;
    return launch_anneal_exact(G, g_diag, b, x0, nullptr, nullptr, 1, n_dim, n_batch, s, spins,
                               diverged, steps, mvms, (cudaStream_t)stream);
}

int il_run_anneals_host(const double* G, const double* g_diag, const double* b, const double* x0,
                        int32_t n_dim, int32_t n_batch, double dt, double p, double a, double zeta,
                        double eps, double e_floor, int32_t f_mvm, int32_t n_steps,
                        double diverge_threshold, int8_t* spins, uint8_t* diverged,
                        int64_t* steps, int64_t* mvms) {
    IL_REQUIRE(n_dim >= 0 && n_batch >= 0, "negative shape");
    const size_t N = (size_t)n_dim, S = 2 * N + 1, B = (size_t)n_batch;
    // one call = one problem (the reference's per-RE granularity): a cached
    // stream and one pinned staging buffer per thread, so the call is one
    // H2D copy, the kernel and one D2H copy
    struct Stage {
        cudaStream_t st = nullptr;
        char* host = nullptr;
        char* dev = nullptr;
        size_t cap = 0;
    };
    static thread_local Stage sg;
    const size_t in_bytes = 8 * (N * N + 2 * N + B * S);
    const size_t out_bytes = B * S + B + 16 * B;
    const size_t need = (in_bytes + out_bytes + 256);
    if (!sg.st) IL_CHECK_CUDA(cudaStreamCreateWithFlags(&sg.st, cudaStreamNonBlocking));
    if (need > sg.cap) {
        if (sg.host) cudaFreeHost(sg.host);
        if (sg.dev) cudaFree(sg.dev);
        sg.host = nullptr;
        sg.dev = nullptr;
        sg.cap = 0;
        IL_CHECK_CUDA(cudaMallocHost((void**)&sg.host, need));
        IL_CHECK_CUDA(cudaMalloc((void**)&sg.dev, need));
        sg.cap = need;
    }
    double* h = reinterpret_cast<double*>(sg.host);
    memcpy(h, G, 8 * N * N);
    memcpy(h + N * N, g_diag, 8 * N);
    memcpy(h + N * N + N, b, 8 * N);
    memcpy(h + N * N + 2 * N, x0, 8 * B * S);
    const double* d = reinterpret_cast<const double*>(sg.dev);
    char* dout = sg.dev + (in_bytes + 127) / 128 * 128;
    char* hout = sg.host + (in_bytes + 127) / 128 * 128;
    int64_t* dsteps = reinterpret_cast<int64_t*>(dout);
    int64_t* dmvms = dsteps + B;
    int8_t* dspins = reinterpret_cast<int8_t*>(dmvms + B);
    uint8_t* ddiv = reinterpret_cast<uint8_t*>(dspins + B * S);
    IL_CHECK_CUDA(cudaMemcpyAsync(sg.dev, sg.host, in_bytes, cudaMemcpyHostToDevice, sg.st));
    int rc = il_run_anneals(d, d + N * N, d + N * N + N, d + N * N + 2 * N, n_dim, n_batch, dt, p,
                            a, zeta, eps, e_floor, f_mvm, n_steps, diverge_threshold, dspins, ddiv,
                            dsteps, dmvms, sg.st);
    if (rc == IL_OK) {
        IL_CHECK_CUDA(cudaMemcpyAsync(hout, dout, out_bytes, cudaMemcpyDeviceToHost, sg.st));
        IL_CHECK_CUDA(cudaStreamSynchronize(sg.st));
        memcpy(steps, hout, 8 * B);
        memcpy(mvms, hout + 8 * B, 8 * B);
        memcpy(spins, hout + 16 * B, B * S);
        memcpy(diverged, hout + 16 * B + B * S, B);
    }
    return rc;
}

int il_derive_seeds(const uint64_t* parts, int32_t n_parts, int64_t n, uint64_t* out,
                    void* stream);
int il_initial_states(const uint64_t* seeds, int64_t n, int32_t S, double amplitude, double* x0,
                      void* stream);

int il_mmse_batch(const double* H, const double* y, const double* noise_var, int64_t P,
                  int32_t n_r, int32_t n_t, int32_t qam_order, uint8_t* x_idx, double* energy,
                  int8_t* status, void* stream) {
    IL_REQUIRE(P >= 0 && n_t >= 1 && n_r >= n_t && n_t <= 32,
               "uplink detection requires 1 <= n_t <= n_r, n_t <= 32");
    Alphabet al;
    int rc = make_qam_alphabet(qam_order, &al);
    if (rc) return rc;
    return launch_mmse(H, y, noise_var, P, n_r, n_t, al, x_idx, energy, status,
                       (cudaStream_t)stream);
}

int il_build_ising_batch(const double* H, const double* y, const uint8_t* guess_idx, int64_t P,
                         int32_t n_r, int32_t n_t, int32_t qam_order, double* G, double* g_diag,
                         double* b, double* offset, double* eps_scale, void* stream) {
    IL_REQUIRE(P >= 0 && n_t >= 1 && n_r >= 1 && n_t <= 32, "invalid shape");
    Alphabet al;
    int rc = alphabet_for(qam_order, &al);
    if (rc) return rc;
    return launch_build_ising(H, y, guess_idx, P, n_r, n_t, al, G, g_diag, b, offset, eps_scale,
                              nullptr, 1.0, 0.0, (cudaStream_t)stream);
}

int il_detect_cim_batch(const double* H, const double* y, const double* noise_var, int64_t P,
                        int32_t n_r, int32_t n_t, int32_t qam_order, const uint64_t* seed,
                        const il_cac_params* prm, uint8_t* x_idx, double* energy, int8_t* source,
                        int32_t* anneal_index, int32_t* diverged_count, void* stream) {
    int rc = validate(prm);
    if (rc) return rc;
    IL_REQUIRE(P >= 0 && n_t >= 1 && n_r >= n_t && n_t <= 32,
               "uplink detection requires 1 <= n_t <= n_r, n_t <= 32");
    IL_REQUIRE(P == 0 || x_idx != nullptr, "x_idx must not be NULL");
    Alphabet al;
    rc = make_qam_alphabet(qam_order, &al);
    if (rc) return rc;
    if (P == 0) return IL_OK;
    cudaStream_t st = (cudaStream_t)stream;
    const int N = 2 * n_t;
    Workspace ws(st);
    double* G = ws.get<double>((size_t)P * N * N, &rc);
    double* g = ws.get<double>((size_t)P * N, &rc);
    double* b = ws.get<double>((size_t)P * N, &rc);
    double* off = ws.get<double>((size_t)P, &rc);
    double* eps = ws.get<double>((size_t)P, &rc);
    uint64_t* base = ws.get<uint64_t>((size_t)P, &rc);
    double* en = energy ? energy : ws.get<double>((size_t)P, &rc);
    int8_t* src = source ? source : ws.get<int8_t>((size_t)P, &rc);
    // the row front end also hands the anneal its operand scale and screen
    // bound (max |G|, sum |G| + sum |b|) so that it need not scan G again
    double* gstats = front_rows_supported(n_r, n_t) ? ws.get<double>((size_t)P * 2, &rc) : nullptr;
    if (rc) return rc;
    const double fixed = prm->eps > 0.0 ? prm->eps : 0.0;
    rc = launch_mmse_ising(H, y, noise_var, P, n_r, n_t, al, x_idx, en, src, G, g, b, off, eps, 1.0,
                           fixed, st, gstats);
    if (rc) return rc;
    rc = launch_base_seeds(seed, P, 0, 0, base, st);  // detector.py:67 derive_seed(seed, 0, 0)
    if (rc) return rc;
    return anneal_and_select(H, y, P, n_r, n_t, al, G, g, b, off, eps, base, prm, x_idx, en, src,
                             anneal_index, diverged_count, st, gstats);
}

int il_residual_batch(const double* H, const double* y, const double* x, int64_t P, int32_t n_r,
                      int32_t n_t, double* energy, void* stream) {
    IL_REQUIRE(P >= 0 && n_r >= 1 && n_t >= 1, "invalid shape");
    return launch_residual(H, y, x, P, n_r, n_t, energy, (cudaStream_t)stream);
}

int il_ml_batch(const double* H, const double* y, int64_t P, int32_t n_r, int32_t n_t,
                int32_t qam_order, uint8_t* x_idx, double* energy, void* stream) {
    IL_REQUIRE(P >= 0 && n_t >= 1 && n_r >= 1, "invalid shape");
    IL_REQUIRE(P == 0 || x_idx, "x_idx must not be NULL");
    Alphabet al;
    int rc = make_qam_alphabet(qam_order, &al);
    if (rc) return rc;
    return launch_ml(H, y, P, n_r, n_t, al, x_idx, energy, (cudaStream_t)stream);
}

int il_ml_llr_batch(const double* H, const double* y, const double* noise_var, int64_t P,
                    int32_t n_r, int32_t n_t, int32_t qam_order, double* llr, void* stream) {
    IL_REQUIRE(P >= 0 && n_t >= 1 && n_r >= 1, "invalid shape");
    IL_REQUIRE(P == 0 || (H && y && llr), "NULL buffer");
    Alphabet al;
    int rc = make_qam_alphabet(qam_order, &al);
    if (rc) return rc;
    return launch_ml_llr(H, y, noise_var, P, n_r, n_t, al, llr, (cudaStream_t)stream);
}

int il_mmse_sic_batch(const double* H, const double* y, const double* noise_var, int64_t P,
                      int32_t n_r, int32_t n_t, int32_t qam_order, uint8_t* x_idx, double* energy,
                      int8_t* status, void* stream) {
    IL_REQUIRE(P >= 0 && n_t >= 1 && n_r >= n_t && n_t <= 32,
               "uplink detection requires 1 <= n_t <= n_r, n_t <= 32");
    IL_REQUIRE(P == 0 || x_idx, "x_idx must not be NULL");
    Alphabet al;
    int rc = make_qam_alphabet(qam_order, &al);
    if (rc) return rc;
    return launch_mmse_sic(H, y, noise_var, P, n_r, n_t, al, x_idx, energy, status,
                           (cudaStream_t)stream);
}

int il_detect_cim_multi_batch(const double* H, const double* y, const double* noise_var,
                              int64_t P, int32_t n_r, int32_t n_t, int32_t qam_order,
                              const uint64_t* seed, const il_cac_params* prm, int32_t n_stages,
                              const int32_t* chains, int32_t n_chains, uint8_t* x_idx,
                              double* energy, int8_t* source, int32_t* anneal_index,
                              int32_t* diverged_count, void* stream) {
    int rc = validate(prm);
    if (rc) return rc;
    IL_REQUIRE(n_stages >= 1, "n_stages must be >= 1");
    IL_REQUIRE(n_chains >= 1 && n_chains <= 8 && chains, "need 1..8 chains");
    for (int c = 0; c < n_chains; ++c)
        IL_REQUIRE(chains[c] == 0 || chains[c] == 1, "chain codes are 0 (mmse) and 1 (mmse_sic)");
    IL_REQUIRE(P >= 0 && n_t >= 1 && n_r >= n_t && n_t <= 32,
               "uplink detection requires 1 <= n_t <= n_r, n_t <= 32");
    IL_REQUIRE(P == 0 || x_idx, "x_idx must not be NULL");
    Alphabet al;
    rc = make_qam_alphabet(qam_order, &al);
    if (rc) return rc;
    if (P == 0) return IL_OK;
    cudaStream_t st = (cudaStream_t)stream;
    const int N = 2 * n_t, nx = 2 * n_t;
    Workspace ws(st);
    uint8_t* bx = ws.get<uint8_t>((size_t)n_chains * P * nx, &rc);    // baselines
    double* be = ws.get<double>((size_t)n_chains * P, &rc);
    int8_t* bst = ws.get<int8_t>((size_t)n_chains * P, &rc);
    int32_t* codes = ws.get<int32_t>((size_t)n_chains, &rc);
    uint8_t* gx = ws.get<uint8_t>((size_t)P * nx, &rc);                // chain guess
    double* ge = ws.get<double>((size_t)P, &rc);
    int8_t* ssrc = ws.get<int8_t>((size_t)P, &rc);
    int32_t* sai = ws.get<int32_t>((size_t)P, &rc);
    int32_t* sdc = ws.get<int32_t>((size_t)P, &rc);
    int32_t* widx = ws.get<int32_t>((size_t)P, &rc);
    double* en = energy ? energy : ws.get<double>((size_t)P, &rc);
    int8_t* src = source ? source : ws.get<int8_t>((size_t)P, &rc);
    int32_t* ai = anneal_index ? anneal_index : ws.get<int32_t>((size_t)P, &rc);
    double* G = ws.get<double>((size_t)P * N * N, &rc);
    double* g = ws.get<double>((size_t)P * N, &rc);
    double* b = ws.get<double>((size_t)P * N, &rc);
    double* off = ws.get<double>((size_t)P, &rc);
    double* eps = ws.get<double>((size_t)P, &rc);
    uint64_t* base = ws.get<uint64_t>((size_t)P, &rc);
    double* gstats = front_rows_supported(n_r, n_t) ? ws.get<double>((size_t)P * 2, &rc) : nullptr;
    if (rc) return rc;
    IL_CHECK_CUDA(cudaMemcpyAsync(codes, chains, sizeof(int32_t) * n_chains,
                                  cudaMemcpyHostToDevice, st));
    for (int c = 0; c < n_chains; ++c) {  // baselines (detector.py:110-111)
        uint8_t* x = bx + (size_t)c * P * nx;
        rc = chains[c] == 0
                 ? launch_mmse(H, y, noise_var, P, n_r, n_t, al, x, be + (size_t)c * P,
                               bst + (size_t)c * P, st)
                 : launch_mmse_sic(H, y, noise_var, P, n_r, n_t, al, x, be + (size_t)c * P,
                                   bst + (size_t)c * P, st);
        if (rc) return rc;
    }
    rc = launch_multi_init(bx, be, bst, codes, n_chains, P, nx, x_idx, en, src, ai, st);
    if (rc) return rc;
    if (diverged_count) IL_CHECK_CUDA(cudaMemsetAsync(diverged_count, 0, sizeof(int32_t) * P, st));
    const double fixed = prm->eps > 0.0 ? prm->eps : 0.0;
    for (int c = 0; c < n_chains; ++c) {  // chains x stages (detector.py:114-131)
        IL_CHECK_CUDA(cudaMemcpyAsync(gx, bx + (size_t)c * P * nx, (size_t)P * nx,
                                      cudaMemcpyDeviceToDevice, st));
        IL_CHECK_CUDA(cudaMemcpyAsync(ge, be + (size_t)c * P, sizeof(double) * P,
                                      cudaMemcpyDeviceToDevice, st));
        IL_CHECK_CUDA(cudaMemsetAsync(widx, 0xff, sizeof(int32_t) * P, st));  // -1
        for (int stage = 0; stage < n_stages; ++stage) {
            rc = launch_build_ising(H, y, gx, P, n_r, n_t, al, G, g, b, off, nullptr, eps, 1.0,
                                    fixed, st, gstats);
            if (rc) return rc;
            rc = launch_base_seeds(seed, P, (uint64_t)c, (uint64_t)stage, base, st);
            if (rc) return rc;
            IL_CHECK_CUDA(cudaMemsetAsync(ssrc, 0, (size_t)P, st));
            rc = anneal_and_select(H, y, P, n_r, n_t, al, G, g, b, off, eps, base, prm, gx, ge,
                                   ssrc, sai, sdc, st, gstats);
            if (rc) return rc;
            rc = launch_multi_stage(sai, P, widx, st);
            if (rc) return rc;
            if (diverged_count) {
                rc = launch_add_i32(sdc, P, diverged_count, st);
                if (rc) return rc;
            }
        }
        rc = launch_multi_combine(gx, ge, widx, P, nx, x_idx, en, src, ai, st);
        if (rc) return rc;
    }
    return IL_OK;
}

int il_precode_vpp_batch(const double* H, const double* u, int64_t P, int32_t n_u, int32_t n_ant,
                         double power, double tau, int32_t n_stages, const uint64_t* seed,
                         const il_cac_params* prm, double* x, double* v, double* unnorm_power,
                         int32_t* diverged_count, void* stream) {
    int rc = validate(prm);
    if (rc) return rc;
    IL_REQUIRE(power > 0, "P must be positive");
    IL_REQUIRE(n_u >= 1 && n_u <= n_ant && n_u <= 32 && n_ant <= 64,
               "downlink precoding requires 1 <= n_u <= n_ant (n_u <= 32, n_ant <= 64)");
    Alphabet al;
    rc = make_lattice_alphabet(n_stages, &al);
    if (rc) return rc;
    if (P == 0) return IL_OK;
    cudaStream_t st = (cudaStream_t)stream;
    const int N = 2 * n_u;
    Workspace ws(st);
    double* W = ws.get<double>((size_t)P * n_ant * n_u * 2, &rc);
    double* Hp = ws.get<double>((size_t)P * n_ant * n_u * 2, &rc);
    double* yt = ws.get<double>((size_t)P * n_ant * 2, &rc);
    double* base_e = ws.get<double>((size_t)P, &rc);
    double* en = ws.get<double>((size_t)P, &rc);
    int8_t* status = ws.get<int8_t>((size_t)P, &rc);
    uint8_t* vidx = ws.get<uint8_t>((size_t)P * 2 * n_u, &rc);
    double* G = ws.get<double>((size_t)P * N * N, &rc);
    double* g = ws.get<double>((size_t)P * N, &rc);
    double* b = ws.get<double>((size_t)P * N, &rc);
    double* off = ws.get<double>((size_t)P, &rc);
    double* eps = ws.get<double>((size_t)P, &rc);
    uint64_t* base = ws.get<uint64_t>((size_t)P, &rc);
    int32_t* stage_div = diverged_count ? ws.get<int32_t>((size_t)P, &rc) : nullptr;
    double* gstats = front_rows_supported(n_ant, n_u) ? ws.get<double>((size_t)P * 2, &rc) : nullptr;
    if (rc) return rc;
    rc = launch_zf_vpp_front(H, u, P, n_u, n_ant, tau, W, yt, Hp, base_e, status, st);
    if (rc) return rc;
    IL_CHECK_CUDA(cudaMemsetAsync(vidx, n_stages, (size_t)P * 2 * n_u, st));  // vhat = 0
    IL_CHECK_CUDA(cudaMemcpyAsync(en, base_e, (size_t)P * 8, cudaMemcpyDeviceToDevice, st));
    if (diverged_count) IL_CHECK_CUDA(cudaMemsetAsync(diverged_count, 0, (size_t)P * 4, st));
    const double fixed = prm->eps > 0.0 ? prm->eps : 0.0;
    for (int stage = 0; stage < n_stages; ++stage) {
        // precoder.py:115-124: _improve_guess(..., derive_seed(seed, 0, stage), eps_gain=1/16)
        rc = launch_build_ising(Hp, yt, vidx, P, n_ant, n_u, al, G, g, b, off, nullptr, eps,
                                0.0625, fixed, st, gstats);
        if (rc) return rc;
        rc = launch_base_seeds(seed, P, 0, (uint64_t)stage, base, st);
        if (rc) return rc;
        rc = anneal_and_select(Hp, yt, P, n_ant, n_u, al, G, g, b, off, eps, base, prm, vidx, en,
                               nullptr, nullptr, stage_div, st, gstats);
        if (rc) return rc;
        if (diverged_count) {
            rc = launch_add_i32(stage_div, P, diverged_count, st);
            if (rc) return rc;
        }
    }
    return launch_vpp_post(W, u, yt, base_e, vidx, P, n_u, n_ant, n_stages, tau, power, x, v,
                           unnorm_power, st);
}

int il_gray_demap(const uint8_t* x_idx, int64_t n_sym, int32_t bits_per_dim, uint8_t* bits,
                  void* stream) {
    return launch_gray_demap(x_idx, n_sym, bits_per_dim, bits, (cudaStream_t)stream);
}

}  // extern "C"
