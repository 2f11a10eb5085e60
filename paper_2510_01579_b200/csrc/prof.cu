// Measurement hooks: kernel-launch counter, per-kernel CUDA-event timing on
// the launching stream, and an FFMA throughput probe (the FP32 roofline
// denominator, which MEASURED_PEAKS.json does not carry).
#include <atomic>
#include <mutex>
#include <vector>

#include "il_internal.cuh"

namespace il {

static std::atomic<long long> g_launches{0};
static std::mutex g_prof_mu;
static bool g_prof_on = false;
struct ProfRec {
    int kind;
    cudaEvent_t a, b;
};
static std::vector<ProfRec> g_prof;

void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

int prof_start(int kind, cudaStream_t st) {
    count_launch();
    std::lock_guard<std::mutex> lk(g_prof_mu);
    if (!g_prof_on) return -1;
    ProfRec r{kind, nullptr, nullptr};
    if (cudaEventCreate(&r.a) != cudaSuccess || cudaEventCreate(&r.b) != cudaSuccess) return -1;
    cudaEventRecord(r.a, st);
    g_prof.push_back(r);
    return (int)g_prof.size() - 1;
}

void prof_stop(int idx, cudaStream_t st) {
    if (idx < 0) return;
    std::lock_guard<std::mutex> lk(g_prof_mu);
    if (idx < (int)g_prof.size()) cudaEventRecord(g_prof[idx].b, st);
}

namespace {
__global__ void k_ffma_probe(float* out, float s, int iters) {
    float a[8];
    const float b = s * threadIdx.x, c = s + 1.f;
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = s * i;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) a[i] = fmaf(a[i], b, c);
    }
    float r = 0.f;
#pragma unroll
    for (int i = 0; i < 8; ++i) r += a[i];
    if (r == 1234.5f) out[0] = r;
}
// The same with packed FFMA2 (two FMAs per instruction), which the anneal's
// Euler update issues: 8 chains x 2 lanes = 16 FMAs per iteration.
__global__ void k_ffma2_probe(float* out, float s, int iters) {
    float2 a[8];
    const float2 b = make_float2(s * threadIdx.x, s * threadIdx.x + 0.25f), c = make_float2(s + 1.f, s + 0.5f);
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = make_float2(s * i, s * i + 0.125f);
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) a[i] = __ffma2_rn(a[i], b, c);
    }
    float r = 0.f;
#pragma unroll
    for (int i = 0; i < 8; ++i) r += a[i].x + a[i].y;
    if (r == 1234.5f) out[0] = r;
}
}  // namespace

}  // namespace il

extern "C" {

long long il_kernel_launches(void) { return il::g_launches.load(); }

void il_profile_begin(void) {
    std::lock_guard<std::mutex> lk(il::g_prof_mu);
    for (auto& r : il::g_prof) {
        cudaEventDestroy(r.a);
        cudaEventDestroy(r.b);
    }
    il::g_prof.clear();
    il::g_prof_on = true;
}

// Sum of event-timed milliseconds per kernel kind (0 front-end, 1 anneal,
// 2 select/decode, 3 other) and launch counts; stops recording.
int il_profile_end(double* ms_by_kind, long long* launches_by_kind, int n_kinds) {
    std::lock_guard<std::mutex> lk(il::g_prof_mu);
    il::g_prof_on = false;
    for (int k = 0; k < n_kinds; ++k) {
        ms_by_kind[k] = 0.0;
        launches_by_kind[k] = 0;
    }
    for (auto& r : il::g_prof) {
        cudaError_t e = cudaEventSynchronize(r.b);
        if (e != cudaSuccess) return il::fail_cuda(e, "il_profile_end");
        float ms = 0.f;
        cudaEventElapsedTime(&ms, r.a, r.b);
        if (r.kind >= 0 && r.kind < n_kinds) {
            ms_by_kind[r.kind] += ms;
            launches_by_kind[r.kind] += 1;
        }
        cudaEventDestroy(r.a);
        cudaEventDestroy(r.b);
    }
    il::g_prof.clear();
    return IL_OK;
}

// Dense FP32 FMA throughput of this GPU (TFLOP/s): the best of `reps`
// launches each of an FFMA and an FFMA2 (packed) probe -- the roofline
// denominator is the faster of the two instructions the anneal issues.
int il_probe_fp32_peak(int reps, double* tflops) {
    float* out = nullptr;
    IL_CHECK_CUDA(cudaMalloc(&out, 4));
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int blocks = sms * 8, threads = 256, iters = 4096;
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    double best = 0.0;
    for (int packed = 0; packed < 2; ++packed) {
        auto launch = [&] {
            if (packed)
                il::k_ffma2_probe<<<blocks, threads>>>(out, 0.5f, iters);
            else
                il::k_ffma_probe<<<blocks, threads>>>(out, 0.5f, iters);
        };
        launch();  // warm-up
        for (int r = 0; r < (reps < 1 ? 1 : reps); ++r) {
            cudaEventRecord(a);
            launch();
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms = 0.f;
            cudaEventElapsedTime(&ms, a, b);
            const double fl = 2.0 * 8.0 * (packed ? 2.0 : 1.0) * iters * (double)blocks * threads;
            if (ms > 0) best = fmax(best, fl / (ms * 1e-3) / 1e12);
        }
    }
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    cudaError_t e = cudaGetLastError();
    cudaFree(out);
    if (e != cudaSuccess) return il::fail_cuda(e, "il_probe_fp32_peak");
    *tflops = best;
    return IL_OK;
}

}  // extern "C"
