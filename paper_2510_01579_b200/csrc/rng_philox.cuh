// Counter-based initial states (CacParams.rng = "philox", IL_RNG_PHILOX):
// Philox4x32-10 (Salmon et al., "Parallel random numbers: as easy as 1, 2,
// 3", SC'11; the generator cuRAND and PyTorch use), written out here and
// checked against cuRAND's curand_Philox4x32_10 and the Random123 known-answer
// vectors by tests/test_rng_host.py.
//
// Draw i of anneal a of a problem with 64-bit base seed s (the same per-
// problem seed the numpy-stream mode keys on, solver.py:182-187) is word i % 4
// of Philox4x32-10(counter = (i / 4, a, kTag, 0), key = (lo32 s, hi32 s)), and
// the state is x0 = fmaf(range, (w >> 8) * 2^-24, lo) in FP32 -- every lane
// computes any draw directly, with no seeding and no sequential stream.  Not
// the reference's numpy streams: parity for this mode is statistical, and
// FP64-exact with rng = "philox" gives the FP64 reference dynamics on the same
// states (the energy gate of north_star "under replayed Philox seeds").
#pragma once
#include <stdint.h>

#ifndef IL_HD
#define IL_HD __host__ __device__ __forceinline__
#endif

namespace il {

constexpr uint32_t kPhiloxM0 = 0xD2511F53u, kPhiloxM1 = 0xCD9E8D57u;
constexpr uint32_t kPhiloxW0 = 0x9E3779B9u, kPhiloxW1 = 0xBB67AE85u;
constexpr uint32_t kPhiloxTag = 0x49534C4Bu;  // counter word 2 of the x0 streams

struct Philox4 {
    uint32_t v[4];
};

IL_HD uint32_t mulhi32(uint32_t a, uint32_t b) {
#ifdef __CUDA_ARCH__
    return __umulhi(a, b);
#else
    return (uint32_t)(((uint64_t)a * b) >> 32);
#endif
}

IL_HD Philox4 philox4x32_10(Philox4 c, uint32_t k0, uint32_t k1) {
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        const uint32_t h0 = mulhi32(kPhiloxM0, c.v[0]), l0 = kPhiloxM0 * c.v[0];
        const uint32_t h1 = mulhi32(kPhiloxM1, c.v[2]), l1 = kPhiloxM1 * c.v[2];
        c = Philox4{{h1 ^ c.v[1] ^ k0, l1, h0 ^ c.v[3] ^ k1, l0}};
        k0 += kPhiloxW0;
        k1 += kPhiloxW1;
    }
    return c;
}

// the four draws 4 blk .. 4 blk + 3 of anneal a: x0 = lo + range * u, FP32
IL_HD void philox_x0_block(uint64_t seed, uint32_t a, uint32_t blk, float lo, float range,
                           float out[4]) {
    const Philox4 w = philox4x32_10(Philox4{{blk, a, kPhiloxTag, 0u}}, (uint32_t)seed,
                                    (uint32_t)(seed >> 32));
#pragma unroll
    for (int q = 0; q < 4; ++q) out[q] = fmaf(range, (float)(w.v[q] >> 8) * 0x1p-24f, lo);
}

}  // namespace il
