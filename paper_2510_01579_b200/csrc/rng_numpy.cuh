// Bit-exact device replay of the NumPy streams the reference draws its
// initial anneal states from:
//   derive_seed(*parts)  = SeedSequence(parts).generate_state(2)      solver.py:137-144
//   default_rng(seed).uniform(lo, hi, S)  (SeedSequence -> PCG64 XSL-RR) solver.py:182-187
//
// Third-party algorithm restated here: NumPy 2.x SeedSequence (pool size 4,
// hashmix/mix constants from numpy/random/bit_generator.pyx) and PCG64
// (pcg64.h: 128-bit LCG, XSL-RR output, setseq seeding), uniform =
// lo + (hi-lo) * ((u64 >> 11) * 2^-53).  Validated against numpy 2.3.5 by
// tests/test_rng.py and the committed fixture tests/golden/seeds.npz.
#pragma once
#include <stdint.h>

#ifndef IL_HD
#define IL_HD __host__ __device__ __forceinline__
#endif

namespace il {

constexpr uint32_t kSsInitA = 0x43b0d7e5u, kSsMultA = 0x931e8875u;
constexpr uint32_t kSsInitB = 0x8b51f9ddu, kSsMultB = 0x58f38dedu;
constexpr uint32_t kSsMixL = 0xca01f9ddu, kSsMixR = 0x4973f715u;

// Words of a non-negative Python int, little-endian 32-bit, at least one.
IL_HD int int_words(uint64_t v, uint32_t* w) {
    w[0] = (uint32_t)v;
    if ((v >> 32) == 0) return 1;
    w[1] = (uint32_t)(v >> 32);
    return 2;
}

IL_HD uint32_t ss_hashmix(uint32_t v, uint32_t& hc) {
    v ^= hc;
    hc *= kSsMultA;
    v *= hc;
    return v ^ (v >> 16);
}
IL_HD uint32_t ss_mix(uint32_t x, uint32_t y) {
    uint32_t r = kSsMixL * x - kSsMixR * y;
    return r ^ (r >> 16);
}

// Entropy pool of SeedSequence(entropy words) (mix_entropy).
IL_HD void ss_pool(const uint32_t* ent, int n, uint32_t pool[4]) {
    uint32_t hc = kSsInitA;
#pragma unroll
    for (int i = 0; i < 4; ++i) pool[i] = ss_hashmix(i < n ? ent[i] : 0u, hc);
#pragma unroll
    for (int s = 0; s < 4; ++s)
#pragma unroll
        for (int d = 0; d < 4; ++d)
            if (s != d) pool[d] = ss_mix(pool[d], ss_hashmix(pool[s], hc));
    for (int s = 4; s < n; ++s)
#pragma unroll
        for (int d = 0; d < 4; ++d) pool[d] = ss_mix(pool[d], ss_hashmix(ent[s], hc));
}

// generate_state(n_words, uint32)
IL_HD void ss_generate(const uint32_t pool[4], uint32_t* out, int n_words) {
    uint32_t hc = kSsInitB;
    for (int i = 0; i < n_words; ++i) {
        uint32_t v = pool[i & 3] ^ hc;
        hc *= kSsMultB;
        v *= hc;
        out[i] = v ^ (v >> 16);
    }
}

// derive_seed(p0, p1, ..., pk) for up to 6 parts (solver.py:137-144).
IL_HD uint64_t derive_seed(const uint64_t* parts, int n_parts) {
    uint32_t ent[12];
    int n = 0;
    for (int i = 0; i < n_parts; ++i) n += int_words(parts[i], ent + n);
    uint32_t pool[4], w[2];
    ss_pool(ent, n, pool);
    ss_generate(pool, w, 2);
    return (uint64_t)w[0] | ((uint64_t)w[1] << 32);
}
IL_HD uint64_t derive_seed2(uint64_t a, uint64_t b) {
    uint64_t p[2] = {a, b};
    return derive_seed(p, 2);
}
IL_HD uint64_t derive_seed3(uint64_t a, uint64_t b, uint64_t c) {
    uint64_t p[3] = {a, b, c};
    return derive_seed(p, 3);
}

// 128-bit unsigned as two 64-bit halves.
struct U128 {
    uint64_t hi, lo;
};

IL_HD U128 mul128(U128 a, U128 b) {
    U128 r;
#ifdef __CUDA_ARCH__
    r.lo = a.lo * b.lo;
    uint64_t h = __umul64hi(a.lo, b.lo);
#else
    unsigned __int128 p = (unsigned __int128)a.lo * b.lo;
    r.lo = (uint64_t)p;
    uint64_t h = (uint64_t)(p >> 64);
#endif
    r.hi = h + a.hi * b.lo + a.lo * b.hi;
    return r;
}
IL_HD U128 add128(U128 a, U128 b) {
    U128 r;
    r.lo = a.lo + b.lo;
    r.hi = a.hi + b.hi + (r.lo < a.lo ? 1u : 0u);
    return r;
}

// PCG64 (NumPy's default bit generator; XSL-RR 128/64).
struct Pcg64 {
    U128 state, inc;

    IL_HD void step() {
        const U128 mult = {0x2360ED051FC65DA4ull, 0x4385DF649FCCF645ull};
        state = add128(mul128(state, mult), inc);
    }
    // default_rng(seed): SeedSequence(seed).generate_state(4, uint64) -> set_seed
    IL_HD void seed_from(uint64_t seed) {
        uint32_t ent[2], pool[4], w[8];
        int n = int_words(seed, ent);
        ss_pool(ent, n, pool);
        ss_generate(pool, w, 8);
        uint64_t u0 = (uint64_t)w[0] | ((uint64_t)w[1] << 32);
        uint64_t u1 = (uint64_t)w[2] | ((uint64_t)w[3] << 32);
        uint64_t u2 = (uint64_t)w[4] | ((uint64_t)w[5] << 32);
        uint64_t u3 = (uint64_t)w[6] | ((uint64_t)w[7] << 32);
        // initstate = (u0, u1), initseq = (u2, u3) as (high, low)
        inc.hi = (u2 << 1) | (u3 >> 63);
        inc.lo = (u3 << 1) | 1u;
        state.hi = 0;
        state.lo = 0;
        step();
        state = add128(state, U128{u0, u1});
        step();
    }
    IL_HD uint64_t next64() {
        step();
        uint64_t x = state.hi ^ state.lo;
        unsigned rot = (unsigned)(state.hi >> 58);
        return (x >> rot) | (x << ((64u - rot) & 63u));
    }
    // uniform(lo, lo + range): lo + range * next_double, no fused multiply-add
    IL_HD double uniform(double lo, double range) {
        double u = (double)(next64() >> 11) * (1.0 / 9007199254740992.0);
#ifdef __CUDA_ARCH__
        return __dadd_rn(lo, __dmul_rn(range, u));
#else
        volatile double t = range * u;
        return lo + t;
#endif
    }
};

}  // namespace il
