// Does legacy mma.sync (HMMA.16816.F32) overlap with packed FP32 (FFMA2) work
// on sm_100a?  Per "period" each warp issues 24 HMMA (4 accumulator chains,
// as the anneal's refresh) and/or 192 FFMA2 (16 independent chains, as its
// two Euler steps).  Modes: 0 FFMA2 only, 1 HMMA only, 2 both in every warp,
// 3 warp-specialised (even warps HMMA, odd warps FFMA2, 2x the work each so
// the total matches mode 2).  Dev tool:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o overlap overlap.cu && ./overlap
#include <cstdio>
#include <cuda_runtime.h>

#define PERIODS 512

__device__ __forceinline__ void mma(float (&d)[4], const unsigned (&a)[4], unsigned b0, unsigned b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
        "{%0,%1,%2,%3};"
        : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

template <int MODE, int MINB>
__global__ void __launch_bounds__(128, MINB) k_ovl(float* out, float s) {
    const int warp = threadIdx.x >> 5;
    bool do_mma = MODE == 1 || MODE == 2 || (MODE == 3 && (warp & 1) == 0);
    bool do_fma = MODE == 0 || MODE == 2 || (MODE == 3 && (warp & 1) == 1);
    const int rep = MODE == 3 ? 2 : 1;
    float2 x[16];
    float acc[4][4];
    unsigned a[4], b0 = __float_as_uint(s) ^ threadIdx.x, b1 = b0 * 3u;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        a[i] = (threadIdx.x * 7u + i) & 0x3bff3bffu;
        acc[i][0] = acc[i][1] = acc[i][2] = acc[i][3] = 0.f;
    }
#pragma unroll
    for (int i = 0; i < 16; ++i) x[i] = make_float2(s * i, s * (i + 1));
    const float2 q = make_float2(0.999f, 0.998f), c = make_float2(s, s);
    for (int p = 0; p < PERIODS; ++p) {
        for (int r = 0; r < rep; ++r) {
            if (do_mma) {
#pragma unroll
                for (int k = 0; k < 6; ++k)
#pragma unroll
                    for (int n = 0; n < 4; ++n) mma(acc[n], a, b0 + k, b1 + n);
            }
            if (do_fma) {
#pragma unroll
                for (int k = 0; k < 12; ++k)
#pragma unroll
                    for (int i = 0; i < 16; ++i) x[i] = __ffma2_rn(x[i], q, c);
            }
        }
    }
    float t = 0.f;
#pragma unroll
    for (int i = 0; i < 16; ++i) t += x[i].x + x[i].y;
#pragma unroll
    for (int n = 0; n < 4; ++n) t += acc[n][0] + acc[n][1] + acc[n][2] + acc[n][3];
    if (t == 1234.5f) out[0] = t;
}

template <int MODE, int MINB>
float run(float* d, int blocks_per_sm) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int blocks = 148 * blocks_per_sm;
    k_ovl<MODE, MINB><<<blocks, 128>>>(d, 1e-3f);
    cudaEventRecord(e0);
    for (int i = 0; i < 5; ++i) k_ovl<MODE, MINB><<<blocks, 128>>>(d, 1e-3f);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    return ms / 5;
}

int main() {
    float* d;
    cudaMalloc(&d, 4);
    for (int bps : {1, 2, 3, 4}) {
        float t0 = run<0, 1>(d, bps), t1 = run<1, 1>(d, bps), t2 = run<2, 1>(d, bps), t3 = run<3, 1>(d, bps);
        // cycles per warp-period per SMSP: ms * clk / (warps per SMSP * periods)
        const double clk = 1.965e6, wps = bps;  // 4 warps per block -> 1 warp per SMSP per block
        auto cyc = [&](float ms) { return ms * clk / (wps * PERIODS); };
        printf("blocks/SM=%d  ffma2-only %.0f  hmma-only %.0f  both/warp %.0f  specialised %.0f  (cycles per warp-period per SMSP; sum %.0f)\n",
               bps, cyc(t0), cyc(t1), cyc(t2), cyc(t3), cyc(t0) + cyc(t1));
    }
    return 0;
}
