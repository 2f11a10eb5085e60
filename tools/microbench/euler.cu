// Microbenchmark of the CIM-CAC Euler update alone (the 64% share of the
// anneal kernel that is not the coupling refresh): how close does the packed
// FP32 update get to the FMA-pipe bound, and what do the e-floor / divergence
// max / packing cost.  Dev tool:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o euler euler.cu && ./euler
#include <cstdio>
#include <cuda_runtime.h>

#define STEPS 2048

struct Sc {
    float alpha, ndt, e_floor;
};

__device__ __forceinline__ float max_nan3(float a, float b, float c) {
    float r;
    asm("max.NaN.f32 %0, %1, %2;" : "=f"(r) : "f"(a), "f"(b));
    asm("max.NaN.f32 %0, %0, %1;" : "+f"(r) : "f"(c));
    return r;
}

// MODE bit 0: divergence max, bit 1: e floor, bit 2: scalar (no f32x2)
template <int NP, int MODE, int MINB>
__global__ void __launch_bounds__(128, MINB) k_euler(float* out, Sc s, float seed) {
    float2 x[NP], e[NP], C[NP];
#pragma unroll
    for (int i = 0; i < NP; ++i) {
        x[i] = make_float2(seed * (i + 1) * 1e-3f + threadIdx.x * 1e-6f, -seed * i * 1e-3f);
        e[i] = make_float2(1.f, 1.f);
        C[i] = make_float2(seed * 1e-4f * i, -seed * 2e-4f);
    }
    float dv = 0.f;
    for (int st = 0; st < STEPS; ++st) {
#pragma unroll
        for (int i = 0; i < NP; ++i) {
            if (MODE & 4) {
                float xs[2] = {x[i].x, x[i].y}, es[2] = {e[i].x, e[i].y}, cs[2] = {C[i].x, C[i].y};
#pragma unroll
                for (int k = 0; k < 2; ++k) {
                    const float x2 = xs[k] * xs[k];
                    if (MODE & 1) dv = fmaxf(dv, x2);
                    const float q = fmaf(s.ndt, x2, s.alpha);
                    xs[k] = fmaf(es[k], cs[k], xs[k] * q);
                    es[k] = es[k] * q;
                    if (MODE & 2) es[k] = fmaxf(es[k], s.e_floor);
                }
                x[i] = make_float2(xs[0], xs[1]);
                e[i] = make_float2(es[0], es[1]);
            } else {
                const float2 x2 = __fmul2_rn(x[i], x[i]);
                if (MODE & 1) dv = max_nan3(dv, x2.x, x2.y);
                const float2 q = __ffma2_rn(make_float2(s.ndt, s.ndt), x2, make_float2(s.alpha, s.alpha));
                const float2 t = __fmul2_rn(x[i], q);
                x[i] = __ffma2_rn(e[i], C[i], t);
                const float2 er = __fmul2_rn(e[i], q);
                e[i] = (MODE & 2) ? make_float2(fmaxf(er.x, s.e_floor), fmaxf(er.y, s.e_floor)) : er;
            }
        }
    }
    float r = dv;
#pragma unroll
    for (int i = 0; i < NP; ++i) r += x[i].x + x[i].y + e[i].x + e[i].y;
    if (r == 1234.5f) out[0] = r;
}

template <int NP, int MODE, int MINB>
void run(const char* name, float* out) {
    int dev = 0, sms = 0, per = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_euler<NP, MODE, MINB>, 128, 0);
    const int blocks = sms * per;
    Sc s{1.01f, -0.02f, 1e-6f};
    k_euler<NP, MODE, MINB><<<blocks, 128>>>(out, s, 0.5f);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a);
    k_euler<NP, MODE, MINB><<<blocks, 128>>>(out, s, 0.5f);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    cudaFuncAttributes fa;
    cudaFuncGetAttributes(&fa, k_euler<NP, MODE, MINB>);
    // FMA-pipe work: 5 packed (= 10 scalar) FP32 ops per pair-step
    const double pair_steps = (double)blocks * 128 * NP * STEPS;
    const double scalar_ops = pair_steps * 10;
    const double peak_ops_per_s = 148.0 * 128 * 1.965e9;  // 128 FP32 lanes/clk/SM
    const double frac = scalar_ops / (ms * 1e-3) / peak_ops_per_s;
    printf("%-28s NP=%2d regs=%3d warps/SM=%2d  %.3f ms  %.1f ns/pair-step/SM  FMA-pipe %.1f%%\n",
           name, NP, fa.numRegs, per * 4, ms, ms * 1e6 / (pair_steps / sms), 100 * frac);
}


// Closer to k_anneal_fast's Euler step: dv per anneal half (4 accumulators),
// e-floor by a per-thread bound, the aux spin, the until_refresh branch with
// a cheap stand-in refresh, and the Kg/nKb constants kept live.
template <int MODE, int MINB>
__global__ void __launch_bounds__(128, MINB) k_real(float* out, Sc s, float seed, int f_mvm) {
    constexpr int NP = 16;
    float2 x[NP], e[NP], C[NP], Kg[4], nKb[4];
#pragma unroll
    for (int i = 0; i < NP; ++i) {
        x[i] = make_float2(seed * (i + 1) * 1e-3f + threadIdx.x * 1e-6f, -seed * i * 1e-3f);
        e[i] = make_float2(1.f, 1.f);
        C[i] = make_float2(seed * 1e-4f * i, -seed * 2e-4f);
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) { Kg[i] = make_float2(seed * i, seed); nKb[i] = make_float2(-seed, seed * i); }
    float dv[2][2] = {{0.f, 0.f}, {0.f, 0.f}};
    float xa = seed * 1e-3f, ea = 1.f, Ca = 0.f, dva = 0.f, e_lb = 1.f;
    int until = 0;
    for (int st = 0; st < STEPS; ++st) {
        if ((MODE & 8) && until == 0) {
            until = f_mvm;
            // stand-in refresh: touch C with the constants (keeps them live)
#pragma unroll
            for (int i = 0; i < NP; ++i) C[i] = __ffma2_rn(Kg[i & 3], x[i], nKb[i & 3]);
        }
#pragma unroll
        for (int i = 0; i < NP; ++i) {
            const float2 x2 = __fmul2_rn(x[i], x[i]);
            dv[i >> 3][i & 1] = max_nan3(dv[i >> 3][i & 1], x2.x, x2.y);
            const float2 q = __ffma2_rn(make_float2(s.ndt, s.ndt), x2, make_float2(s.alpha, s.alpha));
            const float2 t = __fmul2_rn(x[i], q);
            x[i] = __ffma2_rn(e[i], C[i], t);
            e[i] = __fmul2_rn(e[i], q);
        }
        if (MODE & 1) {  // bound floor
            const float dmax = fmaxf(fmaxf(dv[0][0], dv[0][1]), fmaxf(dv[1][0], dv[1][1]));
            const float nxt = e_lb * fmaf(s.ndt, dmax, s.alpha);
            if (nxt >= s.e_floor) e_lb = nxt;
            else {
#pragma unroll
                for (int i = 0; i < NP; ++i) e[i] = make_float2(fmaxf(e[i].x, s.e_floor), fmaxf(e[i].y, s.e_floor));
                e_lb = s.e_floor;
            }
        }
        if (MODE & 2) {  // aux spin
            const float x2 = xa * xa;
            dva = fmaxf(dva, x2);
            const float q = fmaf(s.ndt, x2, s.alpha);
            xa = fmaf(ea, Ca, xa * q);
            ea = fmaxf(ea * q, s.e_floor);
            Ca += 1e-9f;
        }
        --until;
    }
    float r = dva + xa + ea;
#pragma unroll
    for (int i = 0; i < NP; ++i) r += x[i].x + x[i].y + e[i].x + e[i].y;
    r += dv[0][0] + dv[0][1] + dv[1][0] + dv[1][1];
    if (r == 1234.5f) out[0] = r;
}

template <int MODE, int MINB>
void run_real(const char* name, float* out) {
    int dev = 0, sms = 0, per = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_real<MODE, MINB>, 128, 0);
    const int blocks = sms * per;
    Sc s{1.01f, -0.02f, 1e-6f};
    k_real<MODE, MINB><<<blocks, 128>>>(out, s, 0.5f, 2);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a);
    k_real<MODE, MINB><<<blocks, 128>>>(out, s, 0.5f, 2);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    cudaFuncAttributes fa;
    cudaFuncGetAttributes(&fa, k_real<MODE, MINB>);
    const double pair_steps = (double)blocks * 128 * 16 * STEPS;
    const double frac = pair_steps * 10 / (ms * 1e-3) / (148.0 * 128 * 1.965e9);
    printf("%-28s regs=%3d warps/SM=%2d  %.3f ms  FMA-pipe %.1f%%\n", name, fa.numRegs, per * 4, ms, 100 * frac);
}

// Same work as k_real<11>, but the loop body is one refresh period of two
// Euler steps (f_mvm = 2 at compile time): no per-step refresh branch.
template <int MINB>
__global__ void __launch_bounds__(128, MINB) k_period(float* out, Sc s, float seed) {
    constexpr int NP = 16;
    float2 x[NP], e[NP], C[NP], Kg[4], nKb[4];
#pragma unroll
    for (int i = 0; i < NP; ++i) {
        x[i] = make_float2(seed * (i + 1) * 1e-3f + threadIdx.x * 1e-6f, -seed * i * 1e-3f);
        e[i] = make_float2(1.f, 1.f);
        C[i] = make_float2(seed * 1e-4f * i, -seed * 2e-4f);
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) { Kg[i] = make_float2(seed * i, seed); nKb[i] = make_float2(-seed, seed * i); }
    float dv[2][2] = {{0.f, 0.f}, {0.f, 0.f}};
    float xa = seed * 1e-3f, ea = 1.f, Ca = 0.f, dva = 0.f, e_lb = 1.f;
    for (int st = 0; st < STEPS; st += 2) {
#pragma unroll
        for (int i = 0; i < NP; ++i) C[i] = __ffma2_rn(Kg[i & 3], x[i], nKb[i & 3]);
#pragma unroll
        for (int k = 0; k < 2; ++k) {
#pragma unroll
            for (int i = 0; i < NP; ++i) {
                const float2 x2 = __fmul2_rn(x[i], x[i]);
                dv[i >> 3][i & 1] = max_nan3(dv[i >> 3][i & 1], x2.x, x2.y);
                const float2 q = __ffma2_rn(make_float2(s.ndt, s.ndt), x2, make_float2(s.alpha, s.alpha));
                const float2 t = __fmul2_rn(x[i], q);
                x[i] = __ffma2_rn(e[i], C[i], t);
                e[i] = __fmul2_rn(e[i], q);
            }
            const float dmax = fmaxf(fmaxf(dv[0][0], dv[0][1]), fmaxf(dv[1][0], dv[1][1]));
            const float nxt = e_lb * fmaf(s.ndt, dmax, s.alpha);
            if (nxt >= s.e_floor) e_lb = nxt;
            else {
#pragma unroll
                for (int i = 0; i < NP; ++i) e[i] = make_float2(fmaxf(e[i].x, s.e_floor), fmaxf(e[i].y, s.e_floor));
                e_lb = s.e_floor;
            }
            const float x2 = xa * xa;
            dva = fmaxf(dva, x2);
            const float q = fmaf(s.ndt, x2, s.alpha);
            xa = fmaf(ea, Ca, xa * q);
            ea = fmaxf(ea * q, s.e_floor);
            Ca += 1e-9f;
        }
    }
    float r = dva + xa + ea;
#pragma unroll
    for (int i = 0; i < NP; ++i) r += x[i].x + x[i].y + e[i].x + e[i].y;
    r += dv[0][0] + dv[0][1] + dv[1][0] + dv[1][1];
    if (r == 1234.5f) out[0] = r;
}

template <int MINB>
void run_period(const char* name, float* out) {
    int dev = 0, sms = 0, per = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_period<MINB>, 128, 0);
    const int blocks = sms * per;
    Sc s{1.01f, -0.02f, 1e-6f};
    k_period<MINB><<<blocks, 128>>>(out, s, 0.5f);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a);
    k_period<MINB><<<blocks, 128>>>(out, s, 0.5f);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    cudaFuncAttributes fa;
    cudaFuncGetAttributes(&fa, k_period<MINB>);
    const double pair_steps = (double)blocks * 128 * 16 * STEPS;
    const double frac = pair_steps * 10 / (ms * 1e-3) / (148.0 * 128 * 1.965e9);
    printf("%-28s regs=%3d warps/SM=%2d  %.3f ms  FMA-pipe %.1f%%\n", name, fa.numRegs, per * 4, ms, 100 * frac);
}

int main() {
    float* out;
    cudaMalloc(&out, 4);
    run<16, 3, 3>("full (div+floor) minb3", out);
    run<16, 3, 4>("full (div+floor) minb4", out);
    run<16, 3, 2>("full (div+floor) minb2", out);
    run<16, 1, 3>("div only", out);
    run<16, 2, 3>("floor only", out);
    run<16, 0, 3>("bare", out);
    run<16, 7, 3>("full scalar", out);
    run<8, 3, 6>("full NP=8 minb6", out);
    run<8, 3, 4>("full NP=8 minb4", out);
    run<4, 3, 8>("full NP=4 minb8", out);
    run<32, 3, 2>("full NP=32 minb2", out);
    run_real<0, 3>("real: div only", out);
    run_real<1, 3>("real: +bound floor", out);
    run_real<3, 3>("real: +aux", out);
    run_real<11, 3>("real: +refresh branch", out);
    run_real<8, 3>("real: div+branch only", out);
    run_period<3>("period body (f_mvm=2 static)", out);
    return 0;
}
