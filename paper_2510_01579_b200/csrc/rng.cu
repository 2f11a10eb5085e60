// Device entry points for the replayed NumPy seed/stream derivation
// (solver.py:137-144 derive_seed, solver.py:182-187 initial states).
#include "il_internal.cuh"
#include "rng_numpy.cuh"

namespace il {
namespace {

__global__ void k_derive_seeds(const uint64_t* __restrict__ parts, int n_parts, int64_t n,
                               uint64_t* __restrict__ out) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    uint64_t p[6];
    for (int k = 0; k < n_parts; ++k) p[k] = parts[i * n_parts + k];
    out[i] = derive_seed(p, n_parts);
}

__global__ void k_initial_states(const uint64_t* __restrict__ seeds, int64_t n, int S, double lo,
                                 double range, double* __restrict__ x0) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    Pcg64 rng;
    rng.seed_from(seeds[i]);
    for (int k = 0; k < S; ++k) x0[i * S + k] = rng.uniform(lo, range);
}

}  // namespace
}  // namespace il

extern "C" {

int il_derive_seeds(const uint64_t* parts, int32_t n_parts, int64_t n, uint64_t* out,
                    void* stream) {
    IL_REQUIRE(n_parts >= 1 && n_parts <= 6, "n_parts must be in [1, 6]");
    IL_REQUIRE(n >= 0, "negative count");
    if (n == 0) return IL_OK;
    cudaStream_t st = (cudaStream_t)stream;
    IL_LAUNCH(il::kProfOther, st,
              il::k_derive_seeds<<<(unsigned)((n + 127) / 128), 128, 0, st>>>(parts, n_parts, n, out));
    IL_CHECK_CUDA(cudaGetLastError());
    return IL_OK;
}

int il_initial_states(const uint64_t* seeds, int64_t n, int32_t S, double amplitude, double* x0,
                      void* stream) {
    IL_REQUIRE(S >= 0 && n >= 0, "negative shape");
    IL_REQUIRE(amplitude > 0, "init_amplitude must be positive");
    if (n == 0 || S == 0) return IL_OK;
    const double lo = -amplitude, range = amplitude - lo;
    cudaStream_t st = (cudaStream_t)stream;
    IL_LAUNCH(il::kProfOther, st,
              il::k_initial_states<<<(unsigned)((n + 127) / 128), 128, 0, st>>>(seeds, n, S, lo,
                                                                                 range, x0));
    IL_CHECK_CUDA(cudaGetLastError());
    return IL_OK;
}

}  // extern "C"
