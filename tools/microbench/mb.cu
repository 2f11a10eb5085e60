// Microbenchmarks for B200 pipe throughput: FFMA, FFMA2 (f32x2), HFMA2, DFMA,
// mma.sync tf32/f16, LDS.128 broadcast. Used to pick the anneal kernel design.
#include <cstdio>
#include <cuda_runtime.h>
#include <cuda_fp16.h>
#define ITERS 4096
__global__ void k_ffma(float* out, float s) {
  float a[8]; float b = s * threadIdx.x, c = s + 1.f;
  #pragma unroll
  for (int i = 0; i < 8; i++) a[i] = s * i;
  for (int it = 0; it < ITERS; it++) {
    #pragma unroll
    for (int i = 0; i < 8; i++) a[i] = fmaf(a[i], b, c);
  }
  float r = 0; for (int i = 0; i < 8; i++) r += a[i];
  if (r == 1234.5f) out[0] = r;
}
__global__ void k_ffma2(float* out, float s) {
  unsigned long long a[8]; float bb = s * threadIdx.x, cc = s + 1.f;
  unsigned long long b, c;
  asm("mov.b64 %0, {%1,%1};" : "=l"(b) : "f"(bb));
  asm("mov.b64 %0, {%1,%1};" : "=l"(c) : "f"(cc));
  #pragma unroll
  for (int i = 0; i < 8; i++) { float v = s * i; asm("mov.b64 %0, {%1,%1};" : "=l"(a[i]) : "f"(v)); }
  for (int it = 0; it < ITERS; it++) {
    #pragma unroll
    for (int i = 0; i < 8; i++) asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(a[i]) : "l"(b), "l"(c));
  }
  float r = 0; for (int i = 0; i < 8; i++) { float lo, hi; asm("mov.b64 {%0,%1}, %2;" : "=f"(lo), "=f"(hi) : "l"(a[i])); r += lo + hi; }
  if (r == 1234.5f) out[0] = r;
}
__global__ void k_hfma2(float* out, float s) {
  __half2 a[8]; __half2 b = __float2half2_rn(s * threadIdx.x), c = __float2half2_rn(s);
  #pragma unroll
  for (int i = 0; i < 8; i++) a[i] = __float2half2_rn(s * i);
  for (int it = 0; it < ITERS; it++) {
    #pragma unroll
    for (int i = 0; i < 8; i++) a[i] = __hfma2(a[i], b, c);
  }
  float r = 0; for (int i = 0; i < 8; i++) r += __low2float(a[i]);
  if (r == 1234.5f) out[0] = r;
}
__global__ void k_dfma(float* out, float s) {
  double a[8]; double b = s * threadIdx.x, c = s + 1.0;
  #pragma unroll
  for (int i = 0; i < 8; i++) a[i] = s * i;
  for (int it = 0; it < ITERS / 4; it++) {
    #pragma unroll
    for (int i = 0; i < 8; i++) a[i] = fma(a[i], b, c);
  }
  double r = 0; for (int i = 0; i < 8; i++) r += a[i];
  if (r == 1234.5) out[0] = (float)r;
}
// mixed: 6 FFMA + 2 FMNMX per "spin step" (Euler-like)
__global__ void k_mix(float* out, float s) {
  float x[8], e[8]; float m = 0.f; float c = s;
  #pragma unroll
  for (int i = 0; i < 8; i++) { x[i] = s * i; e[i] = 1.f; }
  for (int it = 0; it < ITERS / 4; it++) {
    #pragma unroll
    for (int i = 0; i < 8; i++) {
      float x2 = x[i] * x[i];
      float q = fmaf(-0.02f, x2, 1.01f);
      float r = fmaf(-0.02f, x2, 1.01f + s);
      float t = x[i] * q;
      x[i] = fmaf(e[i], c, t);
      e[i] = fmaxf(e[i] * r, 1e-6f);
      m = fmaxf(m, fabsf(x[i]));
    }
  }
  float r = m; for (int i = 0; i < 8; i++) r += x[i] + e[i];
  if (r == 1234.5f) out[0] = r;
}
__global__ void k_mma_tf32(float* out, float s) {
  unsigned a0 = __float_as_uint(s), a1 = a0 ^ 1, a2 = a0 ^ 2, a3 = a0 ^ 3, b0 = a0 ^ 4, b1 = a0 ^ 5;
  float d[8][4];
  #pragma unroll
  for (int i = 0; i < 8; i++) for (int j = 0; j < 4; j++) d[i][j] = 0.f;
  for (int it = 0; it < ITERS / 8; it++) {
    #pragma unroll
    for (int i = 0; i < 8; i++)
      asm volatile("mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
        : "+f"(d[i][0]), "+f"(d[i][1]), "+f"(d[i][2]), "+f"(d[i][3]) : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
  }
  float r = 0; for (int i = 0; i < 8; i++) for (int j = 0; j < 4; j++) r += d[i][j];
  if (r == 1234.5f) out[0] = r;
}
__global__ void k_mma_f16(float* out, float s) {
  unsigned a0 = __float_as_uint(s) & 0x3bff3bff, a1 = a0 ^ 1, a2 = a0 ^ 2, a3 = a0 ^ 3, b0 = a0 ^ 4, b1 = a0 ^ 5;
  float d[8][4];
  #pragma unroll
  for (int i = 0; i < 8; i++) for (int j = 0; j < 4; j++) d[i][j] = 0.f;
  for (int it = 0; it < ITERS / 8; it++) {
    #pragma unroll
    for (int i = 0; i < 8; i++)
      asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
        : "+f"(d[i][0]), "+f"(d[i][1]), "+f"(d[i][2]), "+f"(d[i][3]) : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
  }
  float r = 0; for (int i = 0; i < 8; i++) for (int j = 0; j < 4; j++) r += d[i][j];
  if (r == 1234.5f) out[0] = r;
}
// LDS.128 broadcast + 4 FFMA per load
__global__ void k_lds(float* out, float s) {
  __shared__ float4 sm[256];
  for (int i = threadIdx.x; i < 256; i += blockDim.x) sm[i] = make_float4(s, s * i, s + i, s - i);
  __syncthreads();
  float acc[4] = {0, 0, 0, 0}; float v = s * threadIdx.x;
  for (int it = 0; it < ITERS / 64; it++) {
    #pragma unroll
    for (int k = 0; k < 64; k++) {
      float4 g = sm[(k + it) & 255];
      acc[0] = fmaf(g.x, v, acc[0]); acc[1] = fmaf(g.y, v, acc[1]);
      acc[2] = fmaf(g.z, v, acc[2]); acc[3] = fmaf(g.w, v, acc[3]);
    }
  }
  float r = acc[0] + acc[1] + acc[2] + acc[3];
  if (r == 1234.5f) out[0] = r;
}
int main() {
  float* out; cudaMalloc(&out, 4);
  int dev; cudaGetDevice(&dev); cudaDeviceProp p; cudaGetDeviceProperties(&p, dev);
  printf("%s SMs=%d clock=%d kHz\n", p.name, p.multiProcessorCount, p.clockRate);
  cudaEvent_t t0, t1; cudaEventCreate(&t0); cudaEventCreate(&t1);
  int blocks = p.multiProcessorCount * 8, threads = 256;
  auto run = [&](const char* name, void (*k)(float*, float), double ops_per_thread, const char* unit) {
    k<<<blocks, threads>>>(out, 0.5f); cudaDeviceSynchronize();
    cudaEventRecord(t0);
    for (int r = 0; r < 5; r++) k<<<blocks, threads>>>(out, 0.5f);
    cudaEventRecord(t1); cudaEventSynchronize(t1);
    float ms; cudaEventElapsedTime(&ms, t0, t1); ms /= 5;
    double tot = ops_per_thread * blocks * threads;
    printf("%-10s %8.3f ms  %8.2f T%s/s\n", name, ms, tot / ms / 1e9, unit);
  };
  run("ffma", k_ffma, 2.0 * 8 * ITERS, "FLOP");
  run("ffma2", k_ffma2, 4.0 * 8 * ITERS, "FLOP");
  run("hfma2", k_hfma2, 4.0 * 8 * ITERS, "FLOP");
  run("dfma", k_dfma, 2.0 * 8 * ITERS / 4, "FLOP");
  run("mix(8ins)", k_mix, 8.0 * 8 * ITERS / 4, "inst");
  run("mma_tf32", k_mma_tf32, 8.0 * ITERS / 8 * 16 * 8 * 8 * 2 / 32, "FLOP");
  run("mma_f16", k_mma_f16, 8.0 * ITERS / 8 * 16 * 8 * 16 * 2 / 32, "FLOP");
  run("lds+4ffma", k_lds, 2.0 * 4 * ITERS, "FLOP");
  cudaError_t e = cudaGetLastError(); printf("err=%s\n", cudaGetErrorString(e));
  return 0;
}
