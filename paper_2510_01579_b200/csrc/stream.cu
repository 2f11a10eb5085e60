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
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <mutex>
#include <vector>

#include "il_internal.cuh"

using namespace il;

#ifndef IL_PIPE_CAP_DIV
#define IL_PIPE_CAP_DIV 8
#endif
#ifndef IL_PIPE_IDLE_CHUNKS
#define IL_PIPE_IDLE_CHUNKS 12
#endif
#ifndef IL_PIPE_TAPER  // halve the last chunks (env ISINGLINK_PIPE_TAPER=2 on, 1 off)
#define IL_PIPE_TAPER 0
#endif
#ifndef IL_PIPE_FIRST_DIV
#define IL_PIPE_FIRST_DIV 48
#endif

namespace {

// Streams and events of the pipeline, created once per device and reused:
// creating 4 streams and 2 x n_chunks events per call cost ~0.4 ms.  Calls
// are serialised by the mutex (the pipeline owns its streams for the call).
struct Streams {
    static constexpr int kMaxComp = 4;
    cudaStream_t in = nullptr, out = nullptr, comp[kMaxComp] = {};
    cudaEvent_t tail = nullptr;  // end of the last enqueued call (streamed slots)
    std::vector<cudaEvent_t> ev;
    int init(int n_events) {
        if (!in)
        {
            for (cudaStream_t* s : {&in, &out})
                IL_CHECK_CUDA(cudaStreamCreateWithFlags(s, cudaStreamNonBlocking));
            for (cudaStream_t& s : comp) IL_CHECK_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
        }
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

// One per-item array moved between host and device: `bytes` per problem.
struct PipeBuf {
    const void* host_in;   // input (H2D) or nullptr
    void* host_out;        // output (D2H) or nullptr
    size_t bytes;
    char* dev = nullptr;
};

// ISINGLINK_PIPE_{FIRST,CAP}_DIV override the ramp (tuning runs)
int env_int(const char* name, int dflt) {
    const char* e = getenv(name);
    const int v = e && *e ? atoi(e) : 0;
    return v > 0 ? v : dflt;
}

// Chunk boundaries: n_chunks > 0 -> equal chunks; otherwise (P >= 4096) a
// ramp: a small first chunk (~P/48, its H2D is the exposed latency) doubling
// up to P/8, so few chunks carry wave tails (streamed slots: 5.54 ms/slot at
// P/8 vs 5.6-5.7 at P/16; one slot at a time the cap is flat).
std::vector<int64_t> chunk_bounds(int64_t P, int n_chunks) {
    static const int cap_div = env_int("ISINGLINK_PIPE_CAP_DIV", IL_PIPE_CAP_DIV);
    static const int first_div = env_int("ISINGLINK_PIPE_FIRST_DIV", IL_PIPE_FIRST_DIV);
    static const bool taper = env_int("ISINGLINK_PIPE_TAPER", IL_PIPE_TAPER + 1) > 1;
    static const int align = env_int("ISINGLINK_PIPE_ALIGN", 0);
    std::vector<int64_t> bounds{0};
    if (n_chunks > 0 || P < 4096) {
        if (n_chunks <= 0) n_chunks = 1;
        n_chunks = (int)std::min<int64_t>(std::min(n_chunks, 64), P);
        int64_t chunk = (P + n_chunks - 1) / n_chunks;
        chunk = (chunk + 7) / 8 * 8;
        while (bounds.back() < P) bounds.push_back(std::min(P, bounds.back() + chunk));
    } else {
        int64_t cap = std::max<int64_t>(P / cap_div, 8);
        int64_t c = std::max<int64_t>(P / first_div, 256);
        if (align > 0) {  // whole anneal waves: first chunk one wave, cap a multiple
            c = align;
            cap = std::max<int64_t>(cap / align, 1) * align;
        }
        while (bounds.back() < P) {
            int64_t cc = align > 0 ? std::min(c, cap) : (std::min(c, cap) + 7) / 8 * 8;
            // taper: the last chunks halve (its anneal tail has no next
            // chunk to overlap with)
            const int64_t rem = P - bounds.back();
            if (taper && rem <= 2 * cap && rem > 512) cc = std::min(cc, (rem / 2 + 7) / 8 * 8);
            bounds.push_back(std::min(P, bounds.back() + cc));
            c *= 2;
        }
    }
    return bounds;
}

// The chunked pipeline: H2D of every input chunk on `in`, compute(o, n, s)
// on alternating compute streams once its inputs landed, D2H of the outputs
// on `out` (enqueued last: a copy into pageable memory blocks the host
// thread and must not delay the enqueue of later chunks).
// done == nullptr: synchronous (returns when the outputs are in host memory);
// otherwise *done receives an event recorded after the last D2H copy and the
// call returns once everything is enqueued (il_pipeline_wait completes it).
template <class F>
int run_pipeline(int64_t P, int n_chunks, std::vector<PipeBuf>& bufs, F&& compute,
                 cudaEvent_t* done = nullptr) {
    static const bool trace = env_int("ISINGLINK_PIPE_TRACE", 0) > 0;
    const auto t_start = std::chrono::steady_clock::now();
    int dev_id = 0;
    IL_CHECK_CUDA(cudaGetDevice(&dev_id));
    IL_REQUIRE(dev_id < 64, "device ordinal out of range");
    std::lock_guard<std::mutex> lock(g_pipe_mu);
    Streams& ss = g_pipe[dev_id];
    // A slot enqueued while the previous one is still on the device (streamed
    // slots) has its copies hidden under that slot's compute anyway: two
    // chunks suffice and cost no ramp (5.12 vs 5.28 ms per 16x16 slot).
    if (n_chunks <= 0 && P >= 4096 && ss.tail && cudaEventQuery(ss.tail) == cudaErrorNotReady)
        n_chunks = 2;
    // an idle device: IL_PIPE_IDLE_CHUNKS equal chunks (12: 5.75 ms per 16x16
    // slot against 5.82 for the ramp, `tools/one_slot_sweep.py`); 0 keeps the ramp
    else if (n_chunks <= 0 && P >= 4096 && IL_PIPE_IDLE_CHUNKS > 0)
        n_chunks = IL_PIPE_IDLE_CHUNKS;
    const std::vector<int64_t> bounds = chunk_bounds(P, n_chunks);
    const int K = (int)bounds.size() - 1;
    static const int n_comp = std::min(Streams::kMaxComp, env_int("ISINGLINK_PIPE_STREAMS", 2));
    int rc = ss.init(std::max(2 * K + 1, n_comp));
    if (rc) return rc;
    for (PipeBuf& b : bufs) {  // stream-ordered on `in`, published by the first event
        if (rc) break;
        rc = pool_alloc((void**)&b.dev, b.bytes * P, ss.in);
    }
    // ISINGLINK_PIPE_TRACE=2: per-chunk device timeline (timing events)
    std::vector<cudaEvent_t> tev;
    const bool timeline = env_int("ISINGLINK_PIPE_TRACE", 0) > 1;
    if (timeline) {
        tev.resize(3 * K + 1);
        for (cudaEvent_t& e : tev) cudaEventCreate(&e);
    }
    if (rc == IL_OK) {
        cudaEvent_t ready = ss.ev[2 * K];
        cudaEventRecord(ready, ss.in);
        if (timeline) cudaEventRecord(tev[3 * K], ss.in);
        for (int k = 0; k < n_comp; ++k) cudaStreamWaitEvent(ss.comp[k], ready, 0);
        cudaStreamWaitEvent(ss.out, ready, 0);
        for (int c = 0; c < K && rc == IL_OK; ++c) {
            const int64_t o = bounds[c], n = bounds[c + 1] - o;
            for (PipeBuf& b : bufs)
                if (b.host_in)
                    cudaMemcpyAsync(b.dev + o * b.bytes, (const char*)b.host_in + o * b.bytes,
                                    n * b.bytes, cudaMemcpyHostToDevice, ss.in);
            cudaEventRecord(ss.ev[2 * c], ss.in);
            if (timeline) cudaEventRecord(tev[3 * c], ss.in);
            cudaStream_t cs = ss.comp[c % n_comp];
            cudaStreamWaitEvent(cs, ss.ev[2 * c], 0);
            if (timeline) cudaEventRecord(tev[3 * c + 1], cs);
            rc = compute(o, n, cs);
            if (rc) break;
            cudaEventRecord(ss.ev[2 * c + 1], cs);
            if (timeline) cudaEventRecord(tev[3 * c + 2], cs);
        }
        for (int c = 0; c < K && rc == IL_OK; ++c) {
            const int64_t o = bounds[c], n = bounds[c + 1] - o;
            cudaStreamWaitEvent(ss.out, ss.ev[2 * c + 1], 0);
            for (PipeBuf& b : bufs)
                if (b.host_out)
                    cudaMemcpyAsync((char*)b.host_out + o * b.bytes, b.dev + o * b.bytes,
                                    n * b.bytes, cudaMemcpyDeviceToHost, ss.out);
        }
    }
    // frees are ordered after every use: join the compute streams into `out`
    for (int k = 0; k < n_comp; ++k) {
        cudaEventRecord(ss.ev[k], ss.comp[k]);
        cudaStreamWaitEvent(ss.out, ss.ev[k], 0);
    }
    for (PipeBuf& b : bufs)
        if (b.dev) cudaFreeAsync(b.dev, ss.out);
    if (!ss.tail) cudaEventCreateWithFlags(&ss.tail, cudaEventDisableTiming);
    if (ss.tail) cudaEventRecord(ss.tail, ss.out);
    const auto t_enq = std::chrono::steady_clock::now();
    if (done && rc == IL_OK) {
        cudaError_t e = cudaEventCreateWithFlags(done, cudaEventDisableTiming);
        if (e == cudaSuccess) e = cudaEventRecord(*done, ss.out);
        if (e == cudaSuccess) return IL_OK;
        rc = fail_cuda(e, "host pipeline (submit)");
    }
    cudaError_t e = cudaStreamSynchronize(ss.out);
    if (trace) {
        const auto t_end = std::chrono::steady_clock::now();
        auto us = [](auto a, auto b) { return std::chrono::duration<double, std::micro>(b - a).count(); };
        fprintf(stderr, "[pipe] P=%lld chunks=%d enqueue %.1f us, total %.1f us\n", (long long)P, K,
                us(t_start, t_enq), us(t_start, t_end));
    }
    if (timeline) {
        cudaDeviceSynchronize();
        for (int c = 0; c < K; ++c) {
            float h = 0, a = 0, b = 0;
            cudaEventElapsedTime(&h, tev[3 * K], tev[3 * c]);
            cudaEventElapsedTime(&a, tev[3 * K], tev[3 * c + 1]);
            cudaEventElapsedTime(&b, tev[3 * K], tev[3 * c + 2]);
            fprintf(stderr, "[pipe] chunk %2d n=%6lld h2d_done %.3f  compute %.3f -> %.3f ms\n", c,
                    (long long)(bounds[c + 1] - bounds[c]), h, a, b);
        }
        for (cudaEvent_t& ev : tev) cudaEventDestroy(ev);
    }
    if (rc == IL_OK && e != cudaSuccess) rc = fail_cuda(e, "host pipeline");
    return rc;
}

}  // namespace

namespace {
int detect_host(const double* H, const double* y, const double* noise_var, int64_t P, int32_t n_r,
                int32_t n_t, int32_t qam_order, const uint64_t* seed, const il_cac_params* prm,
                uint8_t* x_idx, double* energy, int8_t* source, int32_t* anneal_index,
                int32_t* diverged_count, int32_t n_chunks, cudaEvent_t* done,
                uint8_t* bits = nullptr);
}

extern "C" int il_detect_cim_host(const double* H, const double* y, const double* noise_var,
                                  int64_t P, int32_t n_r, int32_t n_t, int32_t qam_order,
                                  const uint64_t* seed, const il_cac_params* prm, uint8_t* x_idx,
                                  double* energy, int8_t* source, int32_t* anneal_index,
                                  int32_t* diverged_count, int32_t n_chunks) {
    return detect_host(H, y, noise_var, P, n_r, n_t, qam_order, seed, prm, x_idx, energy, source,
                       anneal_index, diverged_count, n_chunks, nullptr);
}

extern "C" int il_detect_cim_host_submit(const double* H, const double* y,
                                         const double* noise_var, int64_t P, int32_t n_r,
                                         int32_t n_t, int32_t qam_order, const uint64_t* seed,
                                         const il_cac_params* prm, uint8_t* x_idx, double* energy,
                                         int8_t* source, int32_t* anneal_index,
                                         int32_t* diverged_count, int32_t n_chunks,
                                         void** ticket) {
    IL_REQUIRE(ticket, "ticket must not be NULL");
    *ticket = nullptr;
    cudaEvent_t done = nullptr;
    const int rc = detect_host(H, y, noise_var, P, n_r, n_t, qam_order, seed, prm, x_idx, energy,
                               source, anneal_index, diverged_count, n_chunks, &done);
    if (rc == IL_OK) *ticket = done;  // nullptr when P == 0: nothing to wait for
    return rc;
}

extern "C" int il_detect_cim_bits_host_submit(const double* H, const double* y,
                                              const double* noise_var, int64_t P, int32_t n_r,
                                              int32_t n_t, int32_t qam_order, const uint64_t* seed,
                                              const il_cac_params* prm, uint8_t* bits,
                                              uint8_t* x_idx, double* energy, int8_t* source,
                                              int32_t* anneal_index, int32_t* diverged_count,
                                              int32_t n_chunks, void** ticket) {
    IL_REQUIRE(ticket, "ticket must not be NULL");
    *ticket = nullptr;
    cudaEvent_t done = nullptr;
    const int rc = detect_host(H, y, noise_var, P, n_r, n_t, qam_order, seed, prm, x_idx, energy,
                               source, anneal_index, diverged_count, n_chunks, &done,
                               bits);
    if (rc == IL_OK) *ticket = done;
    return rc;
}

extern "C" int il_pipeline_wait(void* ticket) {
    if (!ticket) return IL_OK;
    cudaEvent_t ev = static_cast<cudaEvent_t>(ticket);
    const cudaError_t e = cudaEventSynchronize(ev);
    cudaEventDestroy(ev);
    if (e != cudaSuccess) return fail_cuda(e, "host pipeline (wait)");
    return IL_OK;
}

namespace {
int detect_host(const double* H, const double* y, const double* noise_var, int64_t P, int32_t n_r,
                int32_t n_t, int32_t qam_order, const uint64_t* seed, const il_cac_params* prm,
                uint8_t* x_idx, double* energy, int8_t* source, int32_t* anneal_index,
                int32_t* diverged_count, int32_t n_chunks, cudaEvent_t* done, uint8_t* bits) {
    IL_REQUIRE(P >= 0 && n_t >= 1 && n_r >= n_t && n_t <= 32,
               "uplink detection requires 1 <= n_t <= n_r, n_t <= 32");
    IL_REQUIRE(P == 0 || (H && y && noise_var && seed && prm && (x_idx || bits)), "NULL buffer");
    int bpd = 0;  // Gray bits per PAM dimension
    if (bits) {
        Alphabet al;
        const int rc = make_qam_alphabet(qam_order, &al);
        if (rc) return rc;
        while ((1 << bpd) < al.m) ++bpd;
    }
    if (P == 0) return IL_OK;
    // outputs with a NULL host pointer stay device scratch (x_idx feeds the
    // demapper; the others are not copied back)
    std::vector<PipeBuf> b = {
        {H, nullptr, sizeof(double) * 2 * n_r * n_t}, {y, nullptr, sizeof(double) * 2 * n_r},
        {noise_var, nullptr, sizeof(double)},         {seed, nullptr, sizeof(uint64_t)},
        {nullptr, x_idx, (size_t)2 * n_t},            {nullptr, energy, sizeof(double)},
        {nullptr, source, 1},                         {nullptr, anneal_index, sizeof(int32_t)},
        {nullptr, diverged_count, sizeof(int32_t)},   {nullptr, bits, (size_t)2 * n_t * bpd}};
    if (!bits) b.pop_back();
    return run_pipeline(P, n_chunks, b, [&](int64_t o, int64_t n, cudaStream_t cs) {
        auto at = [&](int k) { return b[k].dev + o * b[k].bytes; };
        int rc = il_detect_cim_batch((const double*)at(0), (const double*)at(1),
                                     (const double*)at(2), n, n_r, n_t, qam_order,
                                     (const uint64_t*)at(3), prm, (uint8_t*)at(4), (double*)at(5),
                                     (int8_t*)at(6), (int32_t*)at(7), (int32_t*)at(8), cs);
        if (rc == IL_OK && bits)
            rc = launch_gray_demap((const uint8_t*)at(4), n * n_t, bpd, (uint8_t*)at(9), cs);
        return rc;
    }, done);
}
}  // namespace

extern "C" int il_precode_vpp_host(const double* H, const double* u, int64_t P, int32_t n_u,
                                   int32_t n_ant, double power, double tau, int32_t n_stages,
                                   const uint64_t* seed, const il_cac_params* prm, double* x,
                                   double* v, double* unnorm_power, int32_t* diverged_count,
                                   int32_t n_chunks) {
    IL_REQUIRE(P >= 0 && n_u >= 1 && n_u <= n_ant, "downlink precoding requires 1 <= n_u <= n_ant");
    IL_REQUIRE(P == 0 || (H && u && seed && prm && x && v), "NULL buffer");
    if (P == 0) return IL_OK;
    std::vector<PipeBuf> b = {
        {H, nullptr, sizeof(double) * 2 * n_u * n_ant}, {u, nullptr, sizeof(double) * 2 * n_u},
        {seed, nullptr, sizeof(uint64_t)},              {nullptr, x, sizeof(double) * 2 * n_ant},
        {nullptr, v, sizeof(double) * 2 * n_u},         {nullptr, unnorm_power, sizeof(double)},
        {nullptr, diverged_count, sizeof(int32_t)}};
    return run_pipeline(P, n_chunks, b, [&](int64_t o, int64_t n, cudaStream_t cs) {
        auto at = [&](int k) { return b[k].dev + o * b[k].bytes; };
        return il_precode_vpp_batch((const double*)at(0), (const double*)at(1), n, n_u, n_ant,
                                    power, tau, n_stages, (const uint64_t*)at(2), prm,
                                    (double*)at(3), (double*)at(4), (double*)at(5),
                                    (int32_t*)at(6), cs);
    });
}
