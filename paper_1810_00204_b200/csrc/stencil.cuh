// stencil.cuh — compile-time geometry of the 3x3 motion stencil.
// Action / stencil id k = 3(dr+1) + (dc+1); k = 4 is "stay".  Laterals of a moving action are
// its two neighbours on the 8-ring [0,1,2,5,8,7,6,3] (reading R3).
#pragma once
#include <cstdint>

namespace qvts {

__host__ __device__ constexpr int st_dr(int k) { return k / 3 - 1; }
__host__ __device__ constexpr int st_dc(int k) { return k % 3 - 1; }
__host__ __device__ constexpr int ring_at(int i) {
    return i == 0 ? 0 : i == 1 ? 1 : i == 2 ? 2 : i == 3 ? 5 : i == 4 ? 8 : i == 5 ? 7 : i == 6 ? 6 : 3;
}
__host__ __device__ constexpr int ring_pos(int k) {
    return k == 0 ? 0 : k == 1 ? 1 : k == 2 ? 2 : k == 5 ? 3 : k == 8 ? 4 : k == 7 ? 5 : k == 6 ? 6 : 7;
}
__host__ __device__ constexpr int lat1(int k) { return ring_at((ring_pos(k) + 7) % 8); }
__host__ __device__ constexpr int lat2(int k) { return ring_at((ring_pos(k) + 1) % 8); }
// bit of neighbour k (k != 4) in the 8-neighbour occupancy byte m8
__host__ __device__ constexpr int nbit(int k) { return k < 4 ? k : k - 1; }

__host__ __device__ constexpr int mask_count(uint32_t m) {
    return ((m >> 0) & 1) + ((m >> 1) & 1) + ((m >> 2) & 1) + ((m >> 3) & 1) + ((m >> 4) & 1) +
           ((m >> 5) & 1) + ((m >> 6) & 1) + ((m >> 7) & 1) + ((m >> 8) & 1);
}
// stencil id of the j-th action (ascending) of mask m
__host__ __device__ constexpr int mask_action(uint32_t m, int j) {
    int seen = 0;
    for (int k = 0; k < 9; ++k)
        if ((m >> k) & 1) {
            if (seen == j) return k;
            ++seen;
        }
    return -1;
}

}  // namespace qvts

// Dispatch a runtime action mask onto the compiled specialisations (A9, A8, A4; reading R19).
#define QVTS_DISPATCH_MASK(mask, MACRO) \
    switch (mask) {                     \
        case 0x1FF: MACRO(0x1FF); break; \
        case 0x1EF: MACRO(0x1EF); break; \
        case 0x0AA: MACRO(0x0AA); break; \
        default: break;                  \
    }
