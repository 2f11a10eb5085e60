// Legacy mma.sync throughput per instruction kind on sm_100a, alone and mixed
// with packed FP32 work (the anneal refresh's candidates):
//   f16  m16n8k16 (f32 acc)   s8/u8 m16n8k32 (s32 acc)   e4m3 m16n8k32 (f32 acc)
// Per warp-period: 24 MMAs (4 accumulator chains) and/or 192 FFMA2.  Prints
// cycles per warp-period per SMSP.  Dev tool:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mma_kinds mma_kinds.cu && ./mma_kinds
#include <cstdio>
#include <cuda_runtime.h>

#define PERIODS 512

template <int KIND>
__device__ __forceinline__ void mma(float (&d)[4], const unsigned (&a)[4], unsigned b0, unsigned b1) {
    if constexpr (KIND == 0) {
        asm volatile(
            "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
            "{%0,%1,%2,%3};"
            : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
            : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
    } else if constexpr (KIND == 1) {
        int* di = reinterpret_cast<int*>(d);
        asm volatile(
            "mma.sync.aligned.m16n8k32.row.col.s32.s8.s8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
            "{%0,%1,%2,%3};"
            : "+r"(di[0]), "+r"(di[1]), "+r"(di[2]), "+r"(di[3])
            : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
    } else if constexpr (KIND == 2) {
        int* di = reinterpret_cast<int*>(d);
        asm volatile(
            "mma.sync.aligned.m16n8k32.row.col.s32.u8.s8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
            "{%0,%1,%2,%3};"
            : "+r"(di[0]), "+r"(di[1]), "+r"(di[2]), "+r"(di[3])
            : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
    } else {
        asm volatile(
            "mma.sync.aligned.m16n8k32.row.col.f32.e4m3.e4m3.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
            "{%0,%1,%2,%3};"
            : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
            : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
    }
}

template <int KIND, bool DO_MMA, bool DO_FMA>
__global__ void __launch_bounds__(128, 1) k_ovl(float* out, float s) {
    float2 x[16];
    float acc[4][4];
    unsigned a[4], b0 = (__float_as_uint(s) ^ threadIdx.x) & 0x3bff3bffu, b1 = (b0 * 3u) & 0x3bff3bffu;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        a[i] = (threadIdx.x * 7u + i) & 0x3bff3bffu;
        acc[i][0] = acc[i][1] = acc[i][2] = acc[i][3] = 0.f;
    }
#pragma unroll
    for (int i = 0; i < 16; ++i) x[i] = make_float2(s * i, s * (i + 1));
    const float2 q = make_float2(0.999f, 0.998f), c = make_float2(s, s);
    for (int p = 0; p < PERIODS; ++p) {
        if (DO_MMA) {
#pragma unroll
            for (int k = 0; k < 6; ++k)
#pragma unroll
                for (int n = 0; n < 4; ++n) mma<KIND>(acc[n], a, b0 + k, b1 + n);
        }
        if (DO_FMA) {
#pragma unroll
            for (int k = 0; k < 12; ++k)
#pragma unroll
                for (int i = 0; i < 16; ++i) x[i] = __ffma2_rn(x[i], q, c);
        }
    }
    float t = 0.f;
#pragma unroll
    for (int i = 0; i < 16; ++i) t += x[i].x + x[i].y;
#pragma unroll
    for (int n = 0; n < 4; ++n) t += acc[n][0] + acc[n][1] + acc[n][2] + acc[n][3];
    if (t == 1234.5f) out[0] = t;
}

template <int KIND, bool M, bool F>
double cyc(float* d, int bps) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int blocks = 148 * bps;
    k_ovl<KIND, M, F><<<blocks, 128>>>(d, 1e-3f);
    cudaEventRecord(e0);
    for (int i = 0; i < 5; ++i) k_ovl<KIND, M, F><<<blocks, 128>>>(d, 1e-3f);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    int dev;
    cudaGetDevice(&dev);
    int khz;
    cudaDeviceGetAttribute(&khz, cudaDevAttrClockRate, dev);
    return ms / 5 * khz / (bps * PERIODS);
}

template <int KIND>
void row(const char* name, float* d) {
    for (int bps : {1, 3}) {
        const double m = cyc<KIND, true, false>(d, bps), f = cyc<KIND, false, true>(d, bps),
                     b = cyc<KIND, true, true>(d, bps);
        printf("%-6s warps/SMSP=%d  24 mma %.0f  192 ffma2 %.0f  both %.0f  (sum %.0f)\n", name, bps, m, f, b,
               m + f);
    }
}

int main() {
    float* d;
    cudaMalloc(&d, 4);
    row<0>("f16", d);
    row<1>("s8", d);
    row<2>("u8s8", d);
    row<3>("e4m3", d);
    printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
