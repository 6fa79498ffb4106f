// leaf.cu — the leaf level of the QV-tree (SURVEY §8(a) S1+S2+S5): for every leaf parent b (a
// depth-(D-1) belief) and every signature class s, the class sums of the linear predict fields
//   h_0 = b,  h_k(y) = b(y - d_k) + occ(y + d_k) b(y)  (8 move directions, reading B3)
// and of their products with Q'(y, a') = Q_MDP(y, a') - qbar (Eq. 4; reading B1),
// from which k_reduce<leaf> forms M_a[s], P(z|b,a) (Eq. 3 normaliser), R(b,a)
// and every sampled child's Q_MDP value.  Same values as k_hist<leaf> (plan.cu); a
// different schedule:
//
// * one CTA = one PAIR of parents x 128 slot-threads, and every thread carries both parents: the
//   accumulators are fp32 pairs (parent 0, parent 1) updated with packed FFMA2/FADD2
//   (fma.rn.f32x2 with the Q' value as a broadcast scalar operand), so each instruction does the
//   work of two and the per-cell overhead (entry, Q' row, addressing, occupancy bits) is shared;
// * slot-thread t owns ONE wall-signature class in every row band of the grid (class slot ranges
//   fixed for the whole map, build_leaf_bands), so it accumulates across all bands in registers
//   and the class reduction runs once per parent pair: one fp64 record per parent instead of one
//   per (parent, band), and no band-partial round trip through HBM;
// * the CTA walks the bands itself: both parents' band tiles (+1-cell halo) land in shared memory
//   by TMA (cp.async.bulk.tensor over a [beliefs][H][W] tensor map; off-map rows and columns are
//   the copy's zero fill), one elected thread issuing and an mbarrier signalling completion, so the
//   staging costs no load instructions and does not queue in front of the slot stream.  A tile row
//   of width W > 248 is cut into column segments of <= 248 cells (+4 halo columns per side; the
//   TMA box limit is 256), each its own box, so the neighbour offsets stay uniform.
// * each thread's slot stream (entry word, Q' row) is copied 3 steps ahead into a shared-memory
//   ring with its own cp.async groups.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <functional>

#include <cuda.h>
#include <cudaTypedefs.h>

#include "qvts_internal.cuh"
#include "stencil.cuh"

namespace qvts {

namespace {

// packed fp32 pairs (x = parent 0, y = parent 1): d = a * s + c and d = a + c on both lanes
__device__ __forceinline__ float2 ffma2s(float2 a, float s, float2 c) {
    unsigned long long av, sv, cv;
    asm("mov.b64 %0, {%1,%2};" : "=l"(av) : "f"(a.x), "f"(a.y));
    asm("mov.b64 %0, {%1,%1};" : "=l"(sv) : "f"(s));
    asm("mov.b64 %0, {%1,%2};" : "=l"(cv) : "f"(c.x), "f"(c.y));
    asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(cv) : "l"(av), "l"(sv));
    float2 r;
    asm("mov.b64 {%0,%1}, %2;" : "=f"(r.x), "=f"(r.y) : "l"(cv));
    return r;
}
__device__ __forceinline__ float2 fadd2(float2 a, float2 c) {
    unsigned long long av, cv;
    asm("mov.b64 %0, {%1,%2};" : "=l"(av) : "f"(a.x), "f"(a.y));
    asm("mov.b64 %0, {%1,%2};" : "=l"(cv) : "f"(c.x), "f"(c.y));
    asm("add.rn.f32x2 %0, %1, %0;" : "+l"(cv) : "l"(av));
    float2 r;
    asm("mov.b64 {%0,%1}, %2;" : "=f"(r.x), "=f"(r.y) : "l"(cv));
    return r;
}

__host__ __device__ constexpr int dir_k(int di) { return di < 4 ? di : di + 1; }   // direction -> stencil id
__host__ __device__ constexpr bool is_diag(int k) { return k == 0 || k == 2 || k == 6 || k == 8; }
// diagonal directions di in {0, 2, 5, 7} -> accumulator 0..3
__host__ __device__ constexpr int diag_slot(int di) { return di == 0 ? 0 : di == 2 ? 1 : di == 5 ? 2 : 3; }

// tensor memory (TMEM) as per-thread fp64 storage: 32x32b shape, thread i of warp w <-> lane
// 32 (w % 4) + i, consecutive 32-bit columns
__device__ __forceinline__ void tm_ld16(uint32_t ta, uint32_t *v) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
                   "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
                 : "r"(ta));
}
__device__ __forceinline__ void tm_ld4(uint32_t ta, uint32_t *v) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]) : "r"(ta));
}
__device__ __forceinline__ void tm_st16(uint32_t ta, const uint32_t *v) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};"
                 :: "r"(ta), "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]),
                    "r"(v[8]), "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15])
                 : "memory");
}
__device__ __forceinline__ void tm_st4(uint32_t ta, const uint32_t *v) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1,%2,%3,%4};"
                 :: "r"(ta), "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]) : "memory");
}
// the 9 class-mass sums of both parents (18 doubles = 36 columns): read, += fp32 band sums, write
__device__ __forceinline__ void tm_sums(uint32_t ta, uint32_t (&w)[36], bool load) {
    if (load) {
        tm_ld16(ta, w); tm_ld16(ta + 16, w + 16); tm_ld4(ta + 32, w + 32);
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    } else {
        tm_st16(ta, w); tm_st16(ta + 16, w + 16); tm_st4(ta + 32, w + 32);
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    }
}

// shared load at a compile-time byte offset from a 32-bit shared address
template <int OFF>
__device__ __forceinline__ float lds_at(uint32_t addr) {
    float v;
    asm volatile("ld.shared.f32 %0, [%1+%2];" : "=f"(v) : "r"(addr), "n"(OFF));
    return v;
}

constexpr int kLeafRing = 8;            // slot-stream ring depth (steps in flight = kLeafRing - 1)

struct LeafArgs {
    const float *beliefs;
    long long bstride;
    const int32_t *vmap;
    long long nwork;
    const long long *nwork_dev;          // graph-captured step: the parent count on the device
    const LeafBand *bands;
    int nb, nsplit;
    const uint32_t *entries;             // per slot: tile index | m8 << 16
    const float4 *qlist;                 // Q' rows, [step][NAP / 4][slot] float4 per band
    int H, W, TP, TS;
    int nseg, SW, HB, rows;              // column segments, segment width, segment stride, band rows
    int use_tma;                         // 1: stage by TMA (tensor map valid), 0: 4-byte cp.async
    double *part;
    int pstride;
    unsigned long long *skipped;         // (CTA, band) tiles skipped (both parents zero there)
    int cs[17];
};

}  // namespace

template <uint32_t MASK, int TPC>
__global__ void __launch_bounds__(kLeafThreads, 2) k_leaf(LeafArgs a, const __grid_constant__ CUtensorMap tmap) {
    constexpr int NA = mask_count(MASK);
    constexpr int NAP = (NA + 3) & ~3;
    constexpr int NQ4 = NAP / 4;
    constexpr int CB = 1 + 8 + 9 * NA;           // class-binned values per parent (k_hist<leaf> layout)
    constexpr int NV = CB + 4;                   // + the 4 diagonal blocked-mass sums
    constexpr int T = kLeafThreads;
    extern __shared__ __align__(128) float4 smem4[];   // TMA destinations: 128-byte aligned
    float *smem = reinterpret_cast<float *>(smem4);
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
    const long long pair = blockIdx.x / a.nsplit;
    const int split = (int)(blockIdx.x - pair * a.nsplit);
    const long long nwork = a.nwork_dev ? *a.nwork_dev : a.nwork;
    if (2 * pair >= nwork) return;
    const int TP = TPC ? TPC : a.TP;
    const int TS = a.TS;
    const bool has1 = 2 * pair + 1 < nwork;
    const float *__restrict__ bp[2];
#pragma unroll
    for (int p = 0; p < 2; ++p) {
        const long long wp = 2 * pair + (p && has1 ? 1 : 0);
        const long long vv = a.vmap ? (long long)a.vmap[wp] : wp;
        bp[p] = a.beliefs + vv * a.bstride;
    }
    const long long vv0 = a.vmap ? (long long)a.vmap[2 * pair] : 2 * pair;
    const long long vv1 = has1 ? (a.vmap ? (long long)a.vmap[2 * pair + 1] : 2 * pair + 1) : vv0;
    __shared__ alignas(8) unsigned long long s_bar;     // TMA completion barrier
    const uint32_t bar_s = (uint32_t)__cvta_generic_to_shared(&s_bar);
    if (t == 0 && a.use_tma) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(bar_s));
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    uint32_t phase = 0;
    // Per-thread accumulators are band-local (fp32 within one band: ~1/8 of a thread's cells) and
    // folded into running totals in tensor memory at every band end, in band order: the 9
    // class-mass sums (b and the 8 h_k) as fp64 (36 columns), the 72 products and 4 diagonal
    // masses as fp32 pairs (152 columns at A8) -- 256 columns per CTA, two CTAs per SM fill the 512.
    constexpr int NACC = 2 * (9 * NA + 4);               // fp32 columns of F and E
    constexpr int NCH = (NACC + 15) / 16;
    constexpr uint32_t TMC = 48 + 16 * NCH <= 128 ? 128u : 256u;   // allocation: a power of 2
    __shared__ uint32_t s_tmem;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
            (uint32_t)__cvta_generic_to_shared(&s_tmem)), "n"(TMC));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();                                     // the barrier is initialised for every thread
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tm_sum = s_tmem + ((uint32_t)(32 * (warp & 3)) << 16);
    const uint32_t tm_acc = tm_sum + 48;                 // F then E, 2 columns per pair, 16-column chunks
    {
        uint32_t z[36];
#pragma unroll
        for (int i = 0; i < 36; ++i) z[i] = 0u;
        tm_sums(tm_sum, z, false);
#pragma unroll
        for (int c = 0; c < NCH; ++c) tm_st16(tm_acc + 16 * c, z);
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    }

    float2 F[9][NA], S[9], E[4];
#pragma unroll
    for (int f = 0; f < 9; ++f) {
        S[f] = make_float2(0.f, 0.f);
#pragma unroll
        for (int j = 0; j < NA; ++j) F[f][j] = make_float2(0.f, 0.f);
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) E[i] = make_float2(0.f, 0.f);
    // pair i of the F/E accumulators (F row-major, then E)
    auto acc_pair = [&](int i) -> float2 & { return i < 9 * NA ? F[i / NA][i % NA] : E[i - 9 * NA]; };

    const uint32_t tbase = (uint32_t)__cvta_generic_to_shared(smem);
    // the slot-stream ring after the two tiles: Q' rows [ring][NQ4][T] float4, entries [ring][T]
    float4 *qring = reinterpret_cast<float4 *>(smem + 2 * TS);
    uint32_t *ering = reinterpret_cast<uint32_t *>(qring + kLeafRing * NQ4 * T);
    const uint32_t qr_s = (uint32_t)__cvta_generic_to_shared(qring);
    const uint32_t er_s = (uint32_t)__cvta_generic_to_shared(ering);
    const uint32_t TP4 = 4u * (uint32_t)TP, TS4 = 4u * (uint32_t)TS;
    // the 3x3 neighbourhoods of one cell for both parents: nb[i] = (parent 0, parent 1) at
    // offset (i / 3 - 1, i % 3 - 1); 32-bit shared addresses, immediate offsets when TP is static
    auto load_nb = [&](uint32_t e, float2 (&nb)[9]) {
        const uint32_t c0 = tbase + ((e & 0xFFFFu) << 2);
        const uint32_t c1 = c0 + TS4;
        if (TPC) {
            constexpr int R4 = 4 * (TPC ? TPC : 1);
#define QVTS_LNB(I, DR, DC)                                 \
    nb[I].x = lds_at<(DR) * R4 + (DC) * 4>(c0);             \
    nb[I].y = lds_at<(DR) * R4 + (DC) * 4>(c1);
            QVTS_LNB(0, -1, -1) QVTS_LNB(1, -1, 0) QVTS_LNB(2, -1, 1)
            QVTS_LNB(3, 0, -1) QVTS_LNB(4, 0, 0) QVTS_LNB(5, 0, 1)
            QVTS_LNB(6, 1, -1) QVTS_LNB(7, 1, 0) QVTS_LNB(8, 1, 1)
#undef QVTS_LNB
        } else {
            const uint32_t u0 = c0 - TP4, d0 = c0 + TP4, u1 = c1 - TP4, d1 = c1 + TP4;
#define QVTS_LNB(I, A0, A1, DC)                              \
    nb[I].x = lds_at<(DC) * 4>(A0);                          \
    nb[I].y = lds_at<(DC) * 4>(A1);
            QVTS_LNB(0, u0, u1, -1) QVTS_LNB(1, u0, u1, 0) QVTS_LNB(2, u0, u1, 1)
            QVTS_LNB(3, c0, c1, -1) QVTS_LNB(4, c0, c1, 0) QVTS_LNB(5, c0, c1, 1)
            QVTS_LNB(6, d0, d1, -1) QVTS_LNB(7, d0, d1, 0) QVTS_LNB(8, d0, d1, 1)
#undef QVTS_LNB
        }
    };
    // one cell: field 0 = b, fields 1 + d = h_d (d = move direction); diagonal blocked mass
    // (occupancy is not class-constant there) added per cell; orthogonal per class in k_reduce
    auto cell = [&](uint32_t e, const float2 (&nb)[9], const float4 (&qv)[NQ4]) {
        const uint32_t m8 = e >> 16;
        float q[NAP];
#pragma unroll
        for (int h = 0; h < NQ4; ++h) {
            q[4 * h] = qv[h].x; q[4 * h + 1] = qv[h].y; q[4 * h + 2] = qv[h].z; q[4 * h + 3] = qv[h].w;
        }
        const float2 b0 = nb[4];
        // the 4 diagonal fields first (their blocked mass is per cell), then the fields in the
        // order b, orthogonal, diagonal, so no product waits on the add that formed its field;
        // every accumulator still sees the cells in the same order (same values)
        float2 hd[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const int d = i == 0 ? 0 : i == 1 ? 2 : i == 2 ? 5 : 7;
            hd[i] = nb[8 - dir_k(d)];
            if (m8 & (1u << d)) {
                hd[i] = fadd2(b0, hd[i]);
                E[i] = fadd2(b0, E[i]);
            }
        }
        S[0] = fadd2(b0, S[0]);
#pragma unroll
        for (int j = 0; j < NA; ++j) F[0][j] = ffma2s(b0, q[j], F[0][j]);
#pragma unroll
        for (int o = 0; o < 8; ++o) {
            const int d = o < 4 ? (o == 0 ? 1 : o == 1 ? 3 : o == 2 ? 4 : 6) : (o == 4 ? 0 : o == 5 ? 2 : o == 6 ? 5 : 7);
            const float2 h = o < 4 ? nb[8 - dir_k(d)] : hd[o - 4];
            S[1 + d] = fadd2(h, S[1 + d]);
#pragma unroll
            for (int j = 0; j < NA; ++j) F[1 + d][j] = ffma2s(h, q[j], F[1 + d][j]);
        }
    };

    const int b_lo = (int)((long long)split * a.nb / a.nsplit);
    const int b_hi = (int)((long long)(split + 1) * a.nb / a.nsplit);
    for (int band = b_lo; band < b_hi; ++band) {
        const LeafBand bi = a.bands[band];
        const int TH = bi.nrows + 2;
        // stage both parents' band: rows [row0 - 1, row0 + rows + 1) of every column segment
        // (grid columns [s SW - 4, s SW + SW + 4)); rows and columns off the map are zeros
        if (a.use_tma) {
            if (t == 0) {
                // the tiles were last read through the generic proxy (previous band / skip scan)
                asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
                const uint32_t bytes = (uint32_t)(2 * a.nseg * TP * (a.rows + 2) * 4);
                asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(bar_s), "r"(bytes)
                             : "memory");
                for (int p = 0; p < 2; ++p)
                    for (int sg = 0; sg < a.nseg; ++sg) {
                        const uint32_t dst = tbase + 4u * (uint32_t)(p * TS + sg * a.HB);
                        const int c0 = sg * a.SW - 4, c1 = bi.row0 - 1, c2 = (int)(p ? vv1 : vv0);
                        asm volatile(
                            "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
                            " [%0], [%1, {%2, %3, %4}], [%5];\n" ::"r"(dst),
                            "l"(reinterpret_cast<uint64_t>(&tmap)), "r"(c0), "r"(c1), "r"(c2), "r"(bar_s)
                            : "memory");
                    }
                // the next band of both parents into L2 meanwhile (TMA prefetch, no shared memory):
                // its load then waits on L2, not HBM
                if (band + 1 < b_hi) {
                    const int c1n = a.bands[band + 1].row0 - 1;
                    for (int p = 0; p < (has1 ? 2 : 1); ++p)
                        for (int sg = 0; sg < a.nseg; ++sg)
                            asm volatile("cp.async.bulk.prefetch.tensor.3d.L2.global.tile [%0, {%1, %2, %3}];\n" ::"l"(
                                             reinterpret_cast<uint64_t>(&tmap)),
                                         "r"(sg * a.SW - 4), "r"(c1n), "r"((int)(p ? vv1 : vv0))
                                         : "memory");
                }
            }
            asm volatile(
                "{\n .reg .pred P1;\n WAIT_%=:\n"
                " mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
                " @!P1 bra WAIT_%=;\n}\n" ::"r"(bar_s), "r"(phase) : "memory");
            phase ^= 1u;
        } else {
            // generic fallback (rows not 16-byte copyable): 4-byte copies, zero-filled off the map
            const int per = TH * TP;
            for (int i = t; i < 2 * a.nseg * per; i += T) {
                const int ps = i / per, rem = i - ps * per;
                const int p = ps / a.nseg, sg = ps - p * a.nseg;
                const int tr = rem / TP, j = rem - tr * TP;
                const int r = bi.row0 - 1 + tr, c = sg * a.SW - 4 + j;
                const bool ok = (p == 0 || has1) && r >= 0 && r < a.H && c >= 0 && c < a.W;
                const float *src = ok ? bp[p] + (long long)r * a.W + c : bp[0];
                asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;\n" ::"r"(
                                 tbase + 4u * (uint32_t)(p * TS + sg * a.HB + tr * TP + j)),
                             "l"(src), "r"(ok ? 4 : 0));
            }
            asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;\n" ::: "memory");
        }
        __syncthreads();
        // active-tile skipping: both parents hold no mass in this band and
        // its halo -> every term of the band is exactly zero; skip it
        // (bit patterns OR-ed: a -0.0f counts as mass, which only forgoes a skip)
        uint32_t any = 0;
        {
            const uint4 *t4 = reinterpret_cast<const uint4 *>(smem);
            const int n4 = (TH * TP) / 4, off4 = TS / 4, hb4 = a.HB / 4;
            for (int sg = 0; sg < a.nseg; ++sg)
                for (int i = t; i < n4; i += T) {
                    const uint4 v = t4[sg * hb4 + i], w = t4[sg * hb4 + i + off4];
                    any |= (v.x | v.y | v.z | v.w) | (w.x | w.y | w.z | w.w);
                }
        }
        if (!__syncthreads_or(any != 0)) {
            if (t == 0 && a.skipped) atomicAdd(a.skipped, 1ULL);
            continue;           // no shared-memory reads happened after the barrier
        }
        // slot stream: each thread's entry word and Q' row are copied kLeafRing - 1 = 7 steps ahead
        // into a shared-memory ring with its own cp.async groups (no CTA barrier: a thread reads
        // only what it copied), so the L2 latency of the stream is hidden; the next cell's
        // neighbourhoods are loaded before the current cell is accumulated.  Streams carry >= 4
        // trailing padding steps (the zero cell), so the look-ahead needs no bound check.
        // ring slots are compile-time (4-cell unroll = ring depth): slot addresses are immediates
        // off per-thread bases; the global stream pointers advance one step per issue
        static_assert(kLeafRing == 8, "the main loop body covers the ring (two 4-cell halves)");
        const uint32_t *egp = a.entries + bi.slot_off + t;
        // Q' list layout [step][h][slot] float4 (build_qlists): a warp's 16-byte copies of one h
        // are 512 contiguous bytes (the [slot][h] layout fetched every 32-byte sector twice)
        const float4 *qgp = a.qlist + bi.slot_off * NQ4 + t;
        const uint32_t er_t = er_s + 4u * (uint32_t)t, qr_t = qr_s + 16u * (uint32_t)t;
        const uint32_t *ering_t = ering + t;
        const float4 *qring_t = qring + t;
#define QVTS_ISSUE(SLOT)                                                                                 \
    {                                                                                                    \
        asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(er_t + 4u * (SLOT) * T), "l"(egp)); \
        _Pragma("unroll") for (int h = 0; h < NQ4; ++h)                                                   \
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(qr_t + 16u * ((SLOT) * NQ4 + h) * T), \
                         "l"(qgp + h * T));                                                              \
        asm volatile("cp.async.commit_group;\n" ::: "memory");                                           \
        egp += T;                                                                                        \
        qgp += T * NQ4;                                                                                  \
    }
#define QVTS_READY() asm volatile("cp.async.wait_group %0;\n" ::"n"(kLeafRing - 2) : "memory")
#define QVTS_FETCH(SLOT, E, QV)                                                                          \
    {                                                                                                    \
        E = ering_t[(SLOT) * T];                                                                         \
        _Pragma("unroll") for (int h = 0; h < NQ4; ++h) QV[h] = qring_t[((SLOT) * NQ4 + h) * T];         \
    }
        QVTS_ISSUE(0) QVTS_ISSUE(1) QVTS_ISSUE(2) QVTS_ISSUE(3) QVTS_ISSUE(4) QVTS_ISSUE(5) QVTS_ISSUE(6)
        QVTS_READY();
        uint32_t eA, eB;
        float4 qA[NQ4], qB[NQ4];
        float2 nbA[9], nbB[9];
        if constexpr (NA > 8) {
            // A9: the 81 product pairs leave no registers for a second neighbourhood / Q' row in
            // flight, so each cell fetches, loads and accumulates in turn (the co-resident warps
            // cover the shared-memory latency)
            for (int i = 0; i < bi.L; i += 8) {
                QVTS_ISSUE(7) QVTS_READY(); QVTS_FETCH(0, eA, qA) load_nb(eA, nbA); cell(eA, nbA, qA);
                QVTS_ISSUE(0) QVTS_READY(); QVTS_FETCH(1, eA, qA) load_nb(eA, nbA); cell(eA, nbA, qA);
                QVTS_ISSUE(1) QVTS_READY(); QVTS_FETCH(2, eA, qA) load_nb(eA, nbA); cell(eA, nbA, qA);
                QVTS_ISSUE(2) QVTS_READY(); QVTS_FETCH(3, eA, qA) load_nb(eA, nbA); cell(eA, nbA, qA);
                if (i + 4 >= bi.L) break;
                QVTS_ISSUE(3) QVTS_READY(); QVTS_FETCH(4, eA, qA) load_nb(eA, nbA); cell(eA, nbA, qA);
                QVTS_ISSUE(4) QVTS_READY(); QVTS_FETCH(5, eA, qA) load_nb(eA, nbA); cell(eA, nbA, qA);
                QVTS_ISSUE(5) QVTS_READY(); QVTS_FETCH(6, eA, qA) load_nb(eA, nbA); cell(eA, nbA, qA);
                QVTS_ISSUE(6) QVTS_READY(); QVTS_FETCH(7, eA, qA) load_nb(eA, nbA); cell(eA, nbA, qA);
            }
        } else {
        QVTS_FETCH(0, eA, qA)
        load_nb(eA, nbA);
        // cell i: issue step i + 7 into slot (i + 7) & 7, wait for step i + 1, fetch it, load its
        // neighbourhoods, accumulate cell i.  L is a multiple of 4: the 8-cell body may stop halfway.
        for (int i = 0; i < bi.L; i += 8) {
            QVTS_ISSUE(7) QVTS_READY(); QVTS_FETCH(1, eB, qB) load_nb(eB, nbB); cell(eA, nbA, qA);
            QVTS_ISSUE(0) QVTS_READY(); QVTS_FETCH(2, eA, qA) load_nb(eA, nbA); cell(eB, nbB, qB);
            QVTS_ISSUE(1) QVTS_READY(); QVTS_FETCH(3, eB, qB) load_nb(eB, nbB); cell(eA, nbA, qA);
            QVTS_ISSUE(2) QVTS_READY(); QVTS_FETCH(4, eA, qA) load_nb(eA, nbA); cell(eB, nbB, qB);
            if (i + 4 >= bi.L) break;
            QVTS_ISSUE(3) QVTS_READY(); QVTS_FETCH(5, eB, qB) load_nb(eB, nbB); cell(eA, nbA, qA);
            QVTS_ISSUE(4) QVTS_READY(); QVTS_FETCH(6, eA, qA) load_nb(eA, nbA); cell(eB, nbB, qB);
            QVTS_ISSUE(5) QVTS_READY(); QVTS_FETCH(7, eB, qB) load_nb(eB, nbB); cell(eA, nbA, qA);
            QVTS_ISSUE(6) QVTS_READY(); QVTS_FETCH(0, eA, qA) load_nb(eA, nbA); cell(eB, nbB, qB);
        }
        }
#undef QVTS_ISSUE
#undef QVTS_READY
#undef QVTS_FETCH
        asm volatile("cp.async.wait_group 0;\n" ::: "memory");
        {   // this band's fp32 class-mass sums into the fp64 totals
            uint32_t w[36];
            tm_sums(tm_sum, w, true);
#pragma unroll
            for (int i = 0; i < 18; ++i) {
                const int f = i >> 1;
                double d = __hiloint2double((int)w[2 * i + 1], (int)w[2 * i]);
                d += (double)((i & 1) ? S[f].y : S[f].x);
                w[2 * i] = (uint32_t)__double2loint(d);
                w[2 * i + 1] = (uint32_t)__double2hiint(d);
            }
            tm_sums(tm_sum, w, false);
#pragma unroll
            for (int f = 0; f < 9; ++f) S[f] = make_float2(0.f, 0.f);
            // F and E: 8 pairs per 16-column chunk, fp32 adds of the band partials
#pragma unroll
            for (int c = 0; c < NCH; ++c) {
                uint32_t v[16];
                tm_ld16(tm_acc + 16 * c, v);
                asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
                for (int k = 0; k < 8; ++k) {
                    const int i = 8 * c + k;
                    if (i < 9 * NA + 4) {
                        float2 &x = acc_pair(i);
                        const float2 tot = fadd2(make_float2(__uint_as_float(v[2 * k]), __uint_as_float(v[2 * k + 1])), x);
                        v[2 * k] = __float_as_uint(tot.x);
                        v[2 * k + 1] = __float_as_uint(tot.y);
                        x = make_float2(0.f, 0.f);
                    }
                }
                tm_st16(tm_acc + 16 * c, v);
            }
            asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        }
        __syncthreads();   // the tiles are overwritten by the next band
    }

    // class reduction, once per parent pair and one parent at a time: red[v][slot] (fp32) and
    // red64[9][slot] (fp64 class masses), then every output (class, value) sums its class's
    // slot-threads in fixed order in fp64 (4 interleaved sums)
    constexpr int RS = T + 1;
    float *red = smem;
    double *red64 = reinterpret_cast<double *>(smem + ((NV * RS + 3) & ~3));
    const int NOUT = 16 * CB + 8;
#pragma unroll
    for (int p = 0; p < 2; ++p) {
#pragma unroll
        for (int c = 0; c < NCH; ++c) {                   // the F / E totals from tensor memory
            uint32_t v[16];
            tm_ld16(tm_acc + 16 * c, v);
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                const int i = 8 * c + k;
                if (i < 9 * NA + 4) red[(9 + i) * RS + t] = __uint_as_float(v[2 * k + p]);
            }
        }
        {
            uint32_t w[36];
            tm_sums(tm_sum, w, true);
#pragma unroll
            for (int f = 0; f < 9; ++f)
                red64[f * T + t] = __hiloint2double((int)w[2 * (2 * f + p) + 1], (int)w[2 * (2 * f + p)]);
        }
        __syncthreads();
        // record layout of k_hist<leaf>: [class][CB] then 8 blocked-mass values (orthogonal ones 0:
        // k_reduce derives them from the class masses); one record per (parent, split)
        const long long wp = 2 * pair + p;
        for (int oo = t; oo < NOUT && wp < nwork; oo += T) {
            int t0 = 0, t1 = 0, v = 0;
            if (oo < 16 * CB) {
                const int c = oo / CB;
                v = oo - c * CB;
                t0 = a.cs[c];
                t1 = a.cs[c + 1];
            } else {
                const int d = oo - 16 * CB;
                if (d == 0 || d == 2 || d == 5 || d == 7) { v = CB + diag_slot(d); t0 = 0; t1 = T; }
            }
            double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
            int th = t0;
            if (v < 9) {                                    // class masses: fp64 per thread
                const double *rp = red64 + v * T;
                for (; th + 3 < t1; th += 4) {
                    s0 += rp[th];
                    s1 += rp[th + 1];
                    s2 += rp[th + 2];
                    s3 += rp[th + 3];
                }
                for (; th < t1; ++th) s0 += rp[th];
            } else {
                const float *rp = red + v * RS;
                for (; th + 3 < t1; th += 4) {
                    s0 += (double)rp[th];
                    s1 += (double)rp[th + 1];
                    s2 += (double)rp[th + 2];
                    s3 += (double)rp[th + 3];
                }
                for (; th < t1; ++th) s0 += (double)rp[th];
            }
            a.part[(wp * a.nsplit + split) * (long long)a.pstride + oo] = (s0 + s1) + (s2 + s3);
        }
        __syncthreads();                                    // red is rewritten for the next parent
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(s_tmem), "n"(TMC));
}

// ---- host side ------------------------------------------------------------------------------------
static constexpr int kLeafSmemBudget = 112 * 1024;   // two CTAs per SM (2 x (112 + 1) KB <= 228 KB): tiles + ring
static size_t leaf_ring_bytes(int NAP) { return (size_t)kLeafRing * kLeafThreads * (NAP * 4 + 4); }

bool leaf_kernel_supported(const Model &m) {
    const char *ev = std::getenv("QVTS_LEAF_KERNEL");           // read per call (0: the k_hist<leaf> path)
    if (ev && std::atoi(ev) == 0) return false;
    return m.mask == 0x1EF || m.mask == 0x0AA || m.mask == 0x1FF;
}

// CTAs per parent pair: one (all bands), at every level.  Parent-count-independent, so the
// summation order -- and every value -- is the same for any batch, wave or rank count.  Splitting
// the bands over CTAs (a band record per CTA, summed by k_reduce) was measured slower even where
// the level is small: C3 latency 0.367 -> 0.330 ms and a C5 episode batch 11.2 -> 7.3 s with one
// CTA per pair (profiles/r02_leaf_nsplit_ab.json).  QVTS_LEAF_NSPLIT (read per call) overrides it
// for measurement.
int leaf_nsplit(const Model &m, int level) {
    (void)level;
    const char *ev = std::getenv("QVTS_LEAF_NSPLIT");
    if (ev && std::atoi(ev) > 0) return std::min(std::atoi(ev), std::max(1, m.leafb.nb));
    return 1;
}

// Class-fixed band lists.  Bands: as tall as two parents' tiles allow (two CTAs per SM), balanced.
// Slots per class n_c (sum = kLeafThreads): greedy on sum over bands of max_c ceil(count_bc / n_c)
// (the steps the CTA walks), then single-slot moves while they help.  Within each band, class-c
// cells are dealt to the class's slots step by step in raster order; within each warp the 32 cells
// of a step get distinct tile residues mod 32 where the class allows, so a warp's shared loads hit
// 32 distinct banks.
qvts_status build_leaf_bands(Model &m, LeafBands &lb) {
    const int T = kLeafThreads;
    const int H = m.H, W = m.W;
    // column segments of SW cells (a multiple of 4) + 4 halo columns per side: TP = SW + 8 <= 256,
    // the TMA box limit; segment stride HB rounded to 128 bytes (TMA destination alignment)
    const int nseg = (W + 247) / 248;
    const int SW = (((W + nseg - 1) / nseg) + 3) & ~3;
    const int TP = SW + 8;
    auto hb_of = [&](int rows) { return (((rows + 2) * TP) + 31) & ~31; };
    int max_rows = H;
    while (max_rows > 1 && ((long long)2 * nseg * hb_of(max_rows) * 4 + (long long)leaf_ring_bytes(m.NAP) > kLeafSmemBudget ||
                            (long long)nseg * hb_of(max_rows) > 65535 || max_rows + 2 > 256))
        --max_rows;
    if ((long long)2 * nseg * hb_of(max_rows) * 4 + (long long)leaf_ring_bytes(m.NAP) > kLeafSmemBudget ||
        (long long)nseg * hb_of(max_rows) > 65535) {
        set_error("grid too wide for the leaf band tile"); return QVTS_ERR_INVALID_ARG;
    }
    const int nb = (H + max_rows - 1) / max_rows;
    const int rows = (H + nb - 1) / nb;
    lb.nb = nb;
    lb.rows = rows;
    lb.TP = TP;
    lb.nseg = nseg;
    lb.SW = SW;
    lb.HB = hb_of(rows);
    lb.TS = nseg * lb.HB;                    // one parent's tile: nseg segments
    std::vector<std::vector<int>> cls((size_t)nb * 16);
    std::vector<long long> cnt((size_t)nb * 16, 0), tot(16, 0);
    for (int b = 0; b < nb; ++b)
        for (int r = b * rows; r < std::min(H, (b + 1) * rows); ++r)
            for (int c = 0; c < W; ++c) {
                const int x = r * W + c;
                if (m.occ[x]) continue;
                cls[(size_t)b * 16 + m.sig[x]].push_back(x);
                cnt[(size_t)b * 16 + m.sig[x]]++;
                tot[m.sig[x]]++;
            }
    std::vector<int> n(16, 0);
    int used = 0;
    for (int c = 0; c < 16; ++c)
        if (tot[c]) { n[c] = 1; ++used; }
    auto cost = [&](const std::vector<int> &nn) {
        long long s = 0;
        for (int b = 0; b < nb; ++b) {
            long long L = 0;
            for (int c = 0; c < 16; ++c)
                if (nn[c]) L = std::max(L, (cnt[(size_t)b * 16 + c] + nn[c] - 1) / nn[c]);
            s += (L + 3) & ~3;
        }
        return s;
    };
    if (used == 0) { n[0] = T; used = T; }
    while (used < T) {
        long long bestv = -1;
        double bestr = 0.0;
        int bc = -1;
        for (int c = 0; c < 16; ++c) {
            if (!tot[c]) continue;
            n[c]++;
            const long long v = cost(n);
            n[c]--;
            const double r = (double)tot[c] / n[c];
            if (bc < 0 || v < bestv || (v == bestv && r > bestr)) { bestv = v; bestr = r; bc = c; }
        }
        n[bc]++;
        ++used;
    }
    for (bool improved = true; improved;) {          // single-slot moves
        improved = false;
        long long cur = cost(n);
        for (int c = 0; c < 16 && !improved; ++c)
            for (int c2 = 0; c2 < 16 && !improved; ++c2) {
                if (c == c2 || n[c] <= (tot[c] ? 1 : 0) || !tot[c2]) continue;
                n[c]--; n[c2]++;
                const long long v = cost(n);
                if (v < cur) { improved = true; }
                else { n[c]++; n[c2]--; }
            }
    }
    std::vector<int> cls_of(T, -1);
    int t0 = 0;
    for (int c = 0; c < 16; ++c) {
        lb.cs[c] = t0;
        for (int j = 0; j < n[c]; ++j) cls_of[t0 + j] = c;
        t0 += n[c];
    }
    lb.cs[16] = t0;
    lb.h_bands.assign(nb, LeafBand{});
    lb.h_slot_cell.clear();
    std::vector<uint32_t> entries;
    long long off = 0, steps = 0;
    const uint32_t pad_e = (uint32_t)(TP + 1);          // segment 0, row 1, column 1 (grid column -3): zeros
    auto tile_index = [&](int x, int row0) {
        const int r = x / W, c = x % W, sg = c / SW;
        return sg * lb.HB + (r - row0 + 1) * TP + (c - sg * SW + 4);
    };
    for (int b = 0; b < nb; ++b) {
        LeafBand &bi = lb.h_bands[b];
        bi.row0 = b * rows;
        bi.nrows = std::min(rows, H - bi.row0);
        int L = 0;
        for (int c = 0; c < 16; ++c)
            if (n[c]) L = std::max(L, (int)((cnt[(size_t)b * 16 + c] + n[c] - 1) / n[c]));
        L = std::max(4, (L + 3) & ~3);               // the kernel's loop is unrolled by 4 cells
        bi.L = L;
        bi.slot_off = off;
        steps += L;
        const int Lpad = L + 8;                       // the ring reads up to 7 steps ahead
        std::vector<std::vector<int>> bucket(16 * 32);
        std::vector<size_t> head(16 * 32, 0);
        for (int c = 0; c < 16; ++c)
            for (int x : cls[(size_t)b * 16 + c]) {
                const int ti = tile_index(x, bi.row0);
                bucket[c * 32 + (ti & 31)].push_back(x);
            }
        std::vector<uint32_t> e((size_t)Lpad * T, pad_e);
        std::vector<int32_t> sc((size_t)Lpad * T, -1);
        std::vector<int> remc(16);
        for (int c = 0; c < 16; ++c) remc[c] = (int)cls[(size_t)b * 16 + c].size();
        const int pad_res = (int)(pad_e & 31);
        for (int step = 0; step < L; ++step)
            for (int g = 0; g < T / 32; ++g) {
                // slots of this warp that receive a cell (their class still has cells in the band)
                int real[32], nreal = 0;
                bool anypad = false;
                for (int tt = 32 * g; tt < 32 * g + 32; ++tt) {
                    const int c = cls_of[tt];
                    if (c >= 0 && remc[c] > 0) { real[nreal++] = tt; remc[c]--; }
                    else anypad = true;
                }
                // bipartite matching slot -> residue (bank) over the residues the slot's class still
                // has cells in (Kuhn's augmenting paths; most-constrained slots first, fuller buckets
                // tried first); the padding cell's bank is left to the padding slots
                auto left = [&](int c, int r) { return (int)(bucket[c * 32 + r].size() - head[c * 32 + r]); };
                int cand[32][32], ncand[32];
                for (int i = 0; i < nreal; ++i) {
                    const int c = cls_of[real[i]];
                    ncand[i] = 0;
                    for (int r = 0; r < 32; ++r)
                        if (left(c, r) > 0 && !(anypad && r == pad_res)) cand[i][ncand[i]++] = r;
                    std::stable_sort(cand[i], cand[i] + ncand[i], [&](int x, int y) { return left(c, x) > left(c, y); });
                }
                int order[32];
                for (int i = 0; i < nreal; ++i) order[i] = i;
                std::stable_sort(order, order + nreal, [&](int x, int y) { return ncand[x] < ncand[y]; });
                int owner[32], match[32];
                for (int r = 0; r < 32; ++r) owner[r] = -1;
                for (int i = 0; i < nreal; ++i) match[i] = -1;
                for (int oi = 0; oi < nreal; ++oi) {
                    bool seen[32] = {false};
                    std::function<bool(int)> aug = [&](int i) -> bool {
                        for (int k = 0; k < ncand[i]; ++k) {
                            const int r = cand[i][k];
                            if (seen[r]) continue;
                            seen[r] = true;
                            if (owner[r] < 0 || aug(owner[r])) { owner[r] = i; match[i] = r; return true; }
                        }
                        return false;
                    };
                    aug(order[oi]);
                }
                for (int i = 0; i < nreal; ++i) {
                    const int tt = real[i], c = cls_of[tt];
                    int r = match[i];
                    if (r < 0) {                                // no free bank: the fullest bucket
                        int bestn = 0;
                        for (int rr = 0; rr < 32; ++rr)
                            if (left(c, rr) > bestn) { bestn = left(c, rr); r = rr; }
                    }
                    const int x = bucket[c * 32 + r][head[c * 32 + r]++];
                    const int ti = tile_index(x, bi.row0);
                    e[(size_t)step * T + tt] = (uint32_t)ti | ((uint32_t)m.m8[x] << 16);
                    sc[(size_t)step * T + tt] = x;
                }
            }
        entries.insert(entries.end(), e.begin(), e.end());
        lb.h_slot_cell.insert(lb.h_slot_cell.end(), sc.begin(), sc.end());
        off += (long long)Lpad * T;
    }
    lb.total_slots = off;
    lb.steps = steps;
    QVTS_TRY(upload(lb.bands, lb.h_bands));
    QVTS_TRY(upload(lb.entries, entries));
    QVTS_TRY(upload(lb.slot_cell, lb.h_slot_cell));
    return QVTS_OK;
}

// cuTensorMapEncodeTiled through the runtime's driver entry point (no libcuda link)
static PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    static bool tried = false;
    if (!tried) {
        tried = true;
        void *p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
        cudaGetLastError();
    }
    return fn;
}

// The beliefs as a [nbel][H][W] fp32 tensor, box = one column segment of one band (+halo) of one
// belief; false when TMA cannot address them (rows or strides not 16-byte multiples, misaligned)
static bool leaf_tensor_map(const Model &m, const float *beliefs, long long bstride, long long nbel, CUtensorMap *tm) {
    const LeafBands &lb = m.leafb;
    if ((m.W & 3) || (bstride & 3) || (reinterpret_cast<uintptr_t>(beliefs) & 15) || nbel < 1) return false;
    PFN_cuTensorMapEncodeTiled_v12000 enc = tensor_map_encoder();
    if (!enc) return false;
    cuuint64_t dims[3] = {(cuuint64_t)m.W, (cuuint64_t)m.H, (cuuint64_t)nbel};
    cuuint64_t strides[2] = {(cuuint64_t)m.W * 4, (cuuint64_t)bstride * 4};
    cuuint32_t box[3] = {(cuuint32_t)lb.TP, (cuuint32_t)(lb.rows + 2), 1};
    cuuint32_t estr[3] = {1, 1, 1};
    return enc(tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<float *>(beliefs), dims, strides, box, estr,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <uint32_t MASK>
static qvts_status launch_leaf_t(Model &m, const float *beliefs, long long bstride, long long nbel,
                                 const int32_t *vmap, long long nwork, int nsplit, int pstride, long long part_off,
                                 cudaStream_t st, const long long *nwork_dev) {
    constexpr int NA = mask_count(MASK);
    constexpr int NV = 1 + 8 + 9 * NA + 4;
    const LeafBands &lb = m.leafb;
    LeafArgs a;
    a.beliefs = beliefs; a.bstride = bstride; a.vmap = vmap; a.nwork = nwork; a.nwork_dev = nwork_dev;
    a.bands = lb.bands.as<LeafBand>(); a.nb = lb.nb; a.nsplit = nsplit;
    a.entries = lb.entries.as<uint32_t>();
    a.qlist = (m.cur_leaf == QVTS_LEAF_FIB ? lb.qlist_fib : lb.qlist).as<float4>();
    a.H = m.H; a.W = m.W; a.TP = lb.TP; a.TS = lb.TS;
    a.nseg = lb.nseg; a.SW = lb.SW; a.HB = lb.HB; a.rows = lb.rows;
    a.part = m.part.as<double>() + part_off; a.pstride = pstride;
    a.skipped = m.counters.as<unsigned long long>() + 2;
    std::memcpy(a.cs, lb.cs, sizeof(a.cs));
    CUtensorMap tm;
    std::memset(&tm, 0, sizeof(tm));
    const char *ev = std::getenv("QVTS_LEAF_TMA");              // read per call (0: cp.async staging)
    a.use_tma = ((!ev || std::atoi(ev) != 0) && leaf_tensor_map(m, beliefs, bstride, nbel, &tm)) ? 1 : 0;
    const size_t smem = std::max(sizeof(float) * 2 * (size_t)lb.TS + leaf_ring_bytes(m.NAP),
                                 sizeof(float) * ((((size_t)NV * (kLeafThreads + 1)) + 3) & ~(size_t)3) +
                                     sizeof(double) * 9 * kLeafThreads);
    auto kfn = lb.TP == 136 ? k_leaf<MASK, 136> : k_leaf<MASK, 0>;
    QVTS_CUDA(cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    const long long nblocks = ((nwork + 1) / 2) * nsplit;
    if (nblocks > 0x7FFFFFFFLL) { set_error("too many leaf blocks"); return QVTS_ERR_INVALID_ARG; }
    if (nblocks == 0) return QVTS_OK;
    cudaEvent_t e0;
    prof_begin(m, 0, st, &e0);
    kfn<<<(unsigned)nblocks, kLeafThreads, smem, st>>>(a, tm);
    prof_end(m, 0, st, e0);
    QVTS_CUDA(cudaGetLastError());
    m.pstat.leaf_cells += nwork * m.n_free;
    return QVTS_OK;
}

qvts_status launch_leaf(Model &m, const float *beliefs, long long bstride, long long nbel, const int32_t *vmap,
                        long long nwork, int nsplit, int pstride, long long part_off, cudaStream_t st,
                        const long long *nwork_dev) {
    switch (m.mask) {
        case 0x1EF:
            return launch_leaf_t<0x1EF>(m, beliefs, bstride, nbel, vmap, nwork, nsplit, pstride, part_off, st, nwork_dev);
        case 0x0AA:
            return launch_leaf_t<0x0AA>(m, beliefs, bstride, nbel, vmap, nwork, nsplit, pstride, part_off, st, nwork_dev);
        case 0x1FF:
            return launch_leaf_t<0x1FF>(m, beliefs, bstride, nbel, vmap, nwork, nsplit, pstride, part_off, st, nwork_dev);
        default: set_error("leaf kernel: unsupported action set"); return QVTS_ERR_INVALID_ARG;
    }
}

}  // namespace qvts
