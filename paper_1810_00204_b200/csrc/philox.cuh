// philox.cuh — Philox4x32-10 counter-based RNG (Salmon et al., SC'11),
// the library's own device implementation (the oracle carries an independent one).
#pragma once
#include <cstdint>

namespace qvts {

__device__ __forceinline__ uint4 philox4x32_10(uint4 c, uint2 k) {
#pragma unroll
    for (int i = 0; i < 10; ++i) {
        if (i) { k.x += 0x9E3779B9u; k.y += 0xBB67AE85u; }
        const uint32_t hi0 = __umulhi(0xD2511F53u, c.x), lo0 = 0xD2511F53u * c.x;
        const uint32_t hi1 = __umulhi(0xCD9E8D57u, c.z), lo1 = 0xCD9E8D57u * c.z;
        c = make_uint4(hi1 ^ c.y ^ k.x, lo1, hi0 ^ c.w ^ k.y, lo0);
    }
    return c;
}

// Appendix A.4: u = ((w >> 8) + 0.5) 2^-24, exact in fp64, in [2^-25, 1 - 2^-25]
__device__ __forceinline__ double philox_uniform(uint32_t w) { return ((double)(w >> 8) + 0.5) * (1.0 / 16777216.0); }

}  // namespace qvts
