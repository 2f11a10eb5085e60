// Host-side check of csrc/rng_philox.cuh against cuRAND's own Philox4x32-10
// (curand_philox4x32_x.h, compiled here as host code).  Reads lines
// "c0 c1 c2 c3 k0 k1" (hex) from stdin and prints "ours curand" as 8 hex
// words; "x0 seed a blk" prints the four FP32 initial states as hex bits.
#include <stdio.h>
#include <string.h>
#include <inttypes.h>
#include <cuda_runtime.h>
#define QUALIFIERS static inline __host__ __device__
#include <curand_philox4x32_x.h>
#include "../../paper_2510_01579_b200/csrc/rng_philox.cuh"

int main() {
    char kind[16];
    while (scanf("%15s", kind) == 1) {
        if (!strcmp(kind, "p")) {
            unsigned c[4], k[2];
            if (scanf("%x %x %x %x %x %x", &c[0], &c[1], &c[2], &c[3], &k[0], &k[1]) != 6) return 1;
            const il::Philox4 o = il::philox4x32_10(il::Philox4{{c[0], c[1], c[2], c[3]}}, k[0], k[1]);
            const uint4 r = curand_Philox4x32_10(make_uint4(c[0], c[1], c[2], c[3]), make_uint2(k[0], k[1]));
            printf("%08x %08x %08x %08x %08x %08x %08x %08x\n", o.v[0], o.v[1], o.v[2], o.v[3], r.x, r.y,
                   r.z, r.w);
        } else if (!strcmp(kind, "x0")) {
            uint64_t s;
            unsigned a, blk;
            if (scanf("%" SCNu64 " %u %u", &s, &a, &blk) != 3) return 1;
            float out[4];
            il::philox_x0_block(s, a, blk, -0.1f, 0.2f, out);
            for (int q = 0; q < 4; ++q) {
                uint32_t bits;
                memcpy(&bits, &out[q], 4);
                printf("%08x%c", bits, q == 3 ? '\n' : ' ');
            }
        }
    }
    return 0;
}
