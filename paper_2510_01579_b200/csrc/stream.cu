// Host-buffer entry point with a chunked copy/compute pipeline.
//
// il_detect_cim_host takes HOST pointers (the shape of the reference's
// numpy-in / numpy-out call) and streams the slot through the device in
// chunks: the H2D copy of chunk c+1 and the D2H copy of chunk c-1 run on
// their own streams while chunk c is detected, so the PCIe transfer of the
// 200 MB slot (complex128 H) hides under compute.  Consecutive chunks
// alternate between two compute streams so the next chunk's front-end can
// fill SMs while the previous chunk's anneal drains.  Pinned host memory is
// required for the overlap (pageable memory works but the copies then
// serialise with the host thread; pageable outputs only delay the tail).
#include <algorithm>
#include <mutex>
#include <vector>

#include "il_internal.cuh"

using namespace il;

#ifndef IL_PIPE_CAP_DIV
#define IL_PIPE_CAP_DIV 16
#endif

namespace {

// Streams and events of the pipeline, created once per device and reused:
// creating 4 streams and 2 x n_chunks events per call cost ~0.4 ms.  Calls
// are serialised by the mutex (the pipeline owns its streams for the call).
struct Streams {
    cudaStream_t in = nullptr, out = nullptr, comp[2] = {nullptr, nullptr};
    std::vector<cudaEvent_t> ev;
    int init(int n_events) {
        if (!in)
            for (cudaStream_t* s : {&in, &out, &comp[0], &comp[1]})
                IL_CHECK_CUDA(cudaStreamCreateWithFlags(s, cudaStreamNonBlocking));
        while ((int)ev.size() < n_events) {
            cudaEvent_t e;
            IL_CHECK_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
            ev.push_back(e);
        }
        return IL_OK;
    }
};

std::mutex g_pipe_mu;
Streams g_pipe[64];  // per device ordinal

void keep_pool_warm() {
    static bool done = false;
    if (done) return;
    int dev = 0;
    cudaMemPool_t pool;
    if (cudaGetDevice(&dev) == cudaSuccess && cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
        uint64_t thr = UINT64_MAX;  // keep freed workspace for the next call
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
    done = true;
}

}  // namespace

extern "C" int il_detect_cim_host(const double* H, const double* y, const double* noise_var,
                                  int64_t P, int32_t n_r, int32_t n_t, int32_t qam_order,
                                  const uint64_t* seed, const il_cac_params* prm, uint8_t* x_idx,
                                  double* energy, int8_t* source, int32_t* anneal_index,
                                  int32_t* diverged_count, int32_t n_chunks) {
    IL_REQUIRE(P >= 0 && n_t >= 1 && n_r >= n_t && n_t <= 32,
               "uplink detection requires 1 <= n_t <= n_r, n_t <= 32");
    IL_REQUIRE(P == 0 || (H && y && noise_var && seed && prm && x_idx), "NULL buffer");
    if (P == 0) return IL_OK;
    keep_pool_warm();
    // chunk boundaries: n_chunks > 0 -> equal chunks; otherwise (P >= 4096)
    // a ramp: a small first chunk (~P/48, its H2D is the exposed latency)
    // doubling up to P/16, so few chunks carry wave tails
    std::vector<int64_t> bounds{0};
    if (n_chunks > 0 || P < 4096) {
        if (n_chunks <= 0) n_chunks = 1;
        n_chunks = (int)std::min<int64_t>(std::min(n_chunks, 64), P);
        int64_t chunk = (P + n_chunks - 1) / n_chunks;
        chunk = (chunk + 7) / 8 * 8;
        while (bounds.back() < P) bounds.push_back(std::min(P, bounds.back() + chunk));
    } else {
        const int64_t cap = std::max<int64_t>(P / IL_PIPE_CAP_DIV, 8);
        int64_t c = std::max<int64_t>(P / 48, 256);
        while (bounds.back() < P) {
            const int64_t cc = (std::min(c, cap) + 7) / 8 * 8;
            bounds.push_back(std::min(P, bounds.back() + cc));
            c *= 2;
        }
    }
    n_chunks = (int)bounds.size() - 1;

    int dev_id = 0;
    IL_CHECK_CUDA(cudaGetDevice(&dev_id));
    IL_REQUIRE(dev_id < 64, "device ordinal out of range");
    std::lock_guard<std::mutex> lock(g_pipe_mu);
    Streams& ss = g_pipe[dev_id];
    int rc = ss.init(2 * n_chunks + 1);
    if (rc) return rc;
    const size_t hsz = (size_t)n_r * n_t * 2, ysz = (size_t)n_r * 2, xsz = (size_t)n_t * 2;
    // device buffers for the whole slot (stream-ordered on `in`; the other
    // streams are ordered after the allocation through the first event)
    double *dH = nullptr, *dy = nullptr, *ds2 = nullptr, *den = nullptr;
    uint64_t* dseed = nullptr;
    uint8_t* dx = nullptr;
    int8_t* dsrc = nullptr;
    int32_t *dai = nullptr, *ddc = nullptr;
    auto alloc = [&](void** p, size_t bytes) {
        if (rc) return;
        cudaError_t e = cudaMallocAsync(p, bytes ? bytes : 1, ss.in);
        if (e != cudaSuccess) rc = fail_cuda(e, "cudaMallocAsync(il_detect_cim_host)");
    };
    alloc((void**)&dH, sizeof(double) * hsz * P);
    alloc((void**)&dy, sizeof(double) * ysz * P);
    alloc((void**)&ds2, sizeof(double) * P);
    alloc((void**)&dseed, sizeof(uint64_t) * P);
    alloc((void**)&dx, xsz * P);
    alloc((void**)&den, sizeof(double) * P);
    alloc((void**)&dsrc, P);
    alloc((void**)&dai, sizeof(int32_t) * P);
    alloc((void**)&ddc, sizeof(int32_t) * P);
    if (rc == IL_OK) {
        cudaEvent_t ready = ss.ev[2 * n_chunks];
        cudaEventRecord(ready, ss.in);
        cudaStreamWaitEvent(ss.comp[0], ready, 0);
        cudaStreamWaitEvent(ss.comp[1], ready, 0);
        cudaStreamWaitEvent(ss.out, ready, 0);
        for (int c = 0; c < n_chunks && rc == IL_OK; ++c) {
            const int64_t o = bounds[c], n = bounds[c + 1] - o;
            cudaMemcpyAsync(dH + o * hsz, H + o * hsz, sizeof(double) * hsz * n,
                            cudaMemcpyHostToDevice, ss.in);
            cudaMemcpyAsync(dy + o * ysz, y + o * ysz, sizeof(double) * ysz * n,
                            cudaMemcpyHostToDevice, ss.in);
            cudaMemcpyAsync(ds2 + o, noise_var + o, sizeof(double) * n, cudaMemcpyHostToDevice,
                            ss.in);
            cudaMemcpyAsync(dseed + o, seed + o, sizeof(uint64_t) * n, cudaMemcpyHostToDevice,
                            ss.in);
            cudaEventRecord(ss.ev[2 * c], ss.in);
            cudaStream_t cs = ss.comp[c & 1];
            cudaStreamWaitEvent(cs, ss.ev[2 * c], 0);
            rc = il_detect_cim_batch(dH + o * hsz, dy + o * ysz, ds2 + o, n, n_r, n_t, qam_order,
                                     dseed + o, prm, dx + o * xsz, den + o, dsrc + o, dai + o,
                                     ddc + o, cs);
            if (rc) break;
            cudaEventRecord(ss.ev[2 * c + 1], cs);
        }
        // D2H copies are enqueued after every chunk's H2D and compute: a copy
        // into pageable memory blocks the host thread, which must not delay
        // the enqueue of later chunks (the outputs are ~1% of the inputs)
        for (int c = 0; c < n_chunks && rc == IL_OK; ++c) {
            const int64_t o = bounds[c], n = bounds[c + 1] - o;
            cudaStreamWaitEvent(ss.out, ss.ev[2 * c + 1], 0);
            cudaMemcpyAsync(x_idx + o * xsz, dx + o * xsz, xsz * n, cudaMemcpyDeviceToHost, ss.out);
            if (energy)
                cudaMemcpyAsync(energy + o, den + o, sizeof(double) * n, cudaMemcpyDeviceToHost,
                                ss.out);
            if (source) cudaMemcpyAsync(source + o, dsrc + o, n, cudaMemcpyDeviceToHost, ss.out);
            if (anneal_index)
                cudaMemcpyAsync(anneal_index + o, dai + o, sizeof(int32_t) * n,
                                cudaMemcpyDeviceToHost, ss.out);
            if (diverged_count)
                cudaMemcpyAsync(diverged_count + o, ddc + o, sizeof(int32_t) * n,
                                cudaMemcpyDeviceToHost, ss.out);
        }
    }
    // frees are ordered after every use: join the compute streams into `out`
    cudaEvent_t done0 = ss.ev[0], done1 = ss.ev[1];
    cudaEventRecord(done0, ss.comp[0]);
    cudaEventRecord(done1, ss.comp[1]);
    cudaStreamWaitEvent(ss.out, done0, 0);
    cudaStreamWaitEvent(ss.out, done1, 0);
    for (void* p : {(void*)dH, (void*)dy, (void*)ds2, (void*)dseed, (void*)dx, (void*)den,
                    (void*)dsrc, (void*)dai, (void*)ddc})
        if (p) cudaFreeAsync(p, ss.out);
    cudaError_t e = cudaStreamSynchronize(ss.out);
    if (rc == IL_OK && e != cudaSuccess) rc = fail_cuda(e, "il_detect_cim_host");
    return rc;
}
