// philox.cuh -- Philox4x32-10 (Salmon et al., SC'11), device side.
// The counter-based generator named by BASELINE.json north_star; counter layout
// of DESIGN.md R22 / R32 (connectivity gaps (i, n>>2, 4, dst_pop); Poisson (i, t, 2, 0);
// initial V (i, 0, 3, 0)).  Written independently of oracle/ (no shared code).
#pragma once
#include <cstdint>

namespace snn {

struct u32x4 { uint32_t x, y, z, w; };

__device__ __forceinline__ u32x4 philox4x32_10(uint32_t c0, uint32_t c1, uint32_t c2, uint32_t c3,
                                               uint32_t k0, uint32_t k1) {
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        const uint32_t lo0 = 0xD2511F53u * c0;
        const uint32_t hi0 = __umulhi(0xD2511F53u, c0);
        const uint32_t lo1 = 0xCD9E8D57u * c2;
        const uint32_t hi1 = __umulhi(0xCD9E8D57u, c2);
        const uint32_t n0 = hi1 ^ c1 ^ k0;
        const uint32_t n2 = hi0 ^ c3 ^ k1;
        c0 = n0; c1 = lo1; c2 = n2; c3 = lo0;
        k0 += 0x9E3779B9u;
        k1 += 0xBB67AE85u;
    }
    return u32x4{c0, c1, c2, c3};
}

__device__ __forceinline__ uint32_t lane_of(const u32x4 &v, uint32_t k) {
    return k == 0 ? v.x : k == 1 ? v.y : k == 2 ? v.z : v.w;
}

}  // namespace snn
