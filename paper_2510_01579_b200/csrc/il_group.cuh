// Lane groups: GS (8, 16 or 32) consecutive lanes of a warp own one
// problem, lane r of the group owning row r of its matrices.
#pragma once
#include "il_common.cuh"

namespace il {

template <int GS>
struct Grp {
    unsigned mask;  // lanes of this group within the warp
    int r;          // lane within the group (= owned row)
    int base;       // first warp lane of the group
    __device__ Grp() {
        const int lane = threadIdx.x & 31;
        r = lane & (GS - 1);
        base = lane & ~(GS - 1);
        mask = (GS == 32) ? 0xffffffffu : (((1u << GS) - 1u) << base);
    }
    __device__ double sum(double v) const {
#pragma unroll
        for (int o = GS / 2; o > 0; o >>= 1) v = __dadd_rn(v, __shfl_xor_sync(mask, v, o, GS));
        return v;
    }
    // two sums with their shuffle trees interleaved (one tree's latency)
    __device__ void sum2(double& a, double& b) const {
#pragma unroll
        for (int o = GS / 2; o > 0; o >>= 1) {
            const double ta = __shfl_xor_sync(mask, a, o, GS), tb = __shfl_xor_sync(mask, b, o, GS);
            a = __dadd_rn(a, ta);
            b = __dadd_rn(b, tb);
        }
    }
    __device__ double bcast(double v, int src) const { return __shfl_sync(mask, v, src, GS); }
    __device__ cplx bcast(cplx v, int src) const { return {bcast(v.re, src), bcast(v.im, src)}; }
    __device__ void sync() const { __syncwarp(mask); }
};

}  // namespace il
