// leafmma.cu — the leaf level's signature-binned products on the tensor cores (SURVEY §8(a) S1+S2+S5).
//
// For every depth-(D-1) parent b the leaf values need, per wall-signature class s (Eq. 3's
// O(x', z) depends on x' only through s) and per "field" f of the linear predict
// (reading B3: bbar_a = p_stay b + p_int h_a + p_lat (h_l1 + h_l2)),
//     sum_{y in s} f(y)            and      sum_{y in s} f(y) Q'(y, a')     (a' = 0..|A|-1),
// with the fields f = b, g_d(y) = b(y - d_k) (8 directions) and D_d(y) = occ(y + d_k) b(y)
// (4 diagonals; h_d = g_d + D_d; orthogonal blocked mass is class-constant and added in
// k_reduce).  Over the cells of one class this is a dense contraction: rows (parent, field) x
// cells  times  cells x columns (Q'(., a'), 1).  Cells are sorted by class and cut into chunks
// of 16 (the MMA's K), so one mma.sync.m16n8k16 covers 8 parents x 2 fields x 16 cells x 8
// columns.  The A operand is gathered from the staged tiles at the field's shift (no copy of
// the shifted beliefs is ever materialised); B (Q') is a model constant.
//
// Precision: fp16 x fp16 products on the tensor core are exact, but its fp32 accumulation
// truncates (measured, profiles/r01_mma_precision.json: 6e-6 relative over 256 chunks), so the
// MMA accumulates at most kLmFold = 4 chunks before they are folded in fp32 (RN) into the current
// class run; the run joins the class's fp32 total in tensor memory when the class changes, and
// the totals become fp64 in the epilogue.  Operands are split hi + lo:
// b 2^14 = hi + lo (fp16 each, exact to 2^-22 relative), Q' = hi + lo likewise, and the three
// products hi*hi + hi*lo + lo*hi are formed (the lo*lo term is below 2^-22).
//
// One CTA per SM (persistent, 8 warps, ~186 KB of shared memory, all 512 TMEM columns) loops over
// groups of 8 parents and, per group, over the row bands: the next band's tiles stream in with
// cp.async while the current band is multiplied (two smem buffers), and are converted in place to
// {hi, lo} fp16 pairs.  The band's class-sorted chunks are cut into 4 ranges; warps w and w + 4
// (one SM sub-partition, one TMEM lane quarter) walk range w % 4, half 0 multiplying the 4
// diagonal pairs (g_d, D_d) and half 1 the pairs (b, g_1), (g_3, g_4), (g_6, -).  Per-class
// totals accumulate in tensor memory (tcgen05.ld / tcgen05.st, 16 columns per class and half)
// so the registers only hold the current class run.  Every output value is produced by one
// thread in a fixed order: bit-deterministic, and every parent's record is independent of the
// parents it is grouped with.  Output: per parent 4 fp64 records (one per range) in k_hist's
// layout, summed by k_reduce in fixed order (nb = 4).
//
// Status: correct (tests/test_gpu_parity.py::test_leaf_mma_*) but measured slower
// than the scalar leaf k_hist at C4 (plan step 75.7 vs 58.0 ms): mma.sync runs at 0.46 MMA/clk/SM
// on this B200 (profiles/r01_mma_peak.json) and each m16n8k16 needs ~8 shared loads + fragment
// permutes, so the kernel issues ~2.9 warp-instructions per (parent, cell) against the scalar
// kernel's 3.7 but at 42% issue efficiency instead of 74%.  Opt-in: QVTS_LEAF_MMA=1.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>

#include <cuda_fp16.h>

#include "qvts_internal.cuh"
#include "stencil.cuh"

namespace qvts {

constexpr int kLmParents = 8;
constexpr int kLmWarps = 4;                  // records per parent: one per TMEM lane quarter
constexpr int kLmThreads = 2 * kLmWarps * 32;  // two warps per quarter (and per SM sub-partition)
constexpr float kLmScale = 16384.f;          // beliefs are split after scaling by 2^14
constexpr int kLmGuard = 32;                 // zeroed words before the first tile
constexpr int kLmFold = 4;                   // chunks accumulated in the MMA before the fp32 fold

// direction index of the p-th diagonal field (D_d and the m8 bit of occ(y + d_k))
__host__ __device__ constexpr int lm_diag_d(int p) { return p == 0 ? 0 : p == 1 ? 2 : p == 2 ? 5 : 7; }

struct LeafMmaArgs {
    const float *beliefs;
    long long bstride;
    const int32_t *vmap;
    long long nwork;
    const long long *nwork_dev;   // graph-captured plan step: device-side parent count
    const int32_t *skip;
    int H, W, TP, R, nb, ptile, vec16;
    const int32_t *wr;            // [nb][5] chunk range of each warp in the band (class-sorted chunks)
    const uint4 *offs;            // [chunk][4 (t)] byte offsets of K positions 2t, 2t+1, 2t+8, 2t+9; class << 28 in .x
    const uint4 *dmask;           // [chunk][4 (t)] per diagonal: byte e = 0x80 if occ(cell e + d_k)
    const uint4 *qfr;             // [chunk][32 (lane)] B fragments of Q' (hi b0, hi b1, lo b0, lo b1)
    double *part;                 // [parent][4 warps][pstride]
    int pstride;
};

__device__ __forceinline__ uint32_t prmt(uint32_t a, uint32_t b, uint32_t sel) {
    uint32_t r;
    asm("prmt.b32 %0, %1, %2, %3;" : "=r"(r) : "r"(a), "r"(b), "r"(sel));
    return r;
}
__device__ __forceinline__ void lm_mma(float (&c)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3, uint32_t b0,
                                       uint32_t b1) {
    asm("mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                 : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
                 : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}
__device__ __forceinline__ uint32_t lm_split(float b) {
    const float x = b * kLmScale;
    const __half h = __float2half_rn(x);
    const __half l = __float2half_rn(x - __half2float(h));
    return (uint32_t)__half_as_ushort(h) | ((uint32_t)__half_as_ushort(l) << 16);
}

// two words at once (f16x2 conversions): {hi(x0) | lo(x0) << 16, hi(x1) | lo(x1) << 16}
__device__ __forceinline__ uint2 lm_split2(float b0, float b1) {
    const float2 x = make_float2(b0 * kLmScale, b1 * kLmScale);
    const __half2 h = __float22half2_rn(x);
    const float2 hf = __half22float2(h);
    const __half2 l = __float22half2_rn(make_float2(x.x - hf.x, x.y - hf.y));
    const uint32_t hu = *reinterpret_cast<const uint32_t *>(&h), lu = *reinterpret_cast<const uint32_t *>(&l);
    return make_uint2(prmt(hu, lu, 0x5410), prmt(hu, lu, 0x7632));
}

// ---- TMEM: 16 consecutive fp32 columns of this thread's lane --------------------------------
#define LM_R16(v) "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), \
    "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
#define LM_W16(v) "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]), \
    "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15])
__device__ __forceinline__ void tm_ld16(uint32_t taddr, uint32_t (&v)[16]) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                 : LM_R16(v) : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tm_st16(uint32_t taddr, const uint32_t (&v)[16]) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};"
                 :: "r"(taddr), LM_W16(v) : "memory");
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
}

// Stage (cp.async) the 8 parents' band tiles into the buffer at smem byte address sbase: warp w
// copies tile rows w, w + 4, ... (row = parent x tile row), lanes stride the columns.
__device__ __forceinline__ void lm_stage(const LeafMmaArgs &a, uint32_t sbase, long long group, int band, long long nwork) {
    const int row0 = band * a.R;
    const int TH = a.R + 2;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int pp = 0; pp < kLmParents; ++pp) {
        const long long wp = group * kLmParents + pp;
        const bool pv = wp < nwork;
        const float *bp = a.beliefs + (pv ? (a.vmap ? (long long)a.vmap[wp] : wp) * a.bstride : 0);
        for (int tr = warp; tr < TH; tr += kLmThreads / 32) {
            const int r = row0 - 1 + tr;
            const bool ok = pv && r >= 0 && r < a.H;
            const float *row = ok ? bp + (long long)r * a.W : a.beliefs;
            const uint32_t dst = sbase + 4u * (uint32_t)(pp * a.ptile + tr * a.TP + 4);
            if (a.vec16) {
                for (int c4 = lane; 4 * c4 < a.W; c4 += 32)
                    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(dst + 16u * c4),
                                 "l"(ok ? row + 4 * c4 : row), "r"(ok ? 16 : 0));
            } else {
                for (int c = lane; c < a.W; c += 32)
                    asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;\n" ::"r"(dst + 4u * c),
                                 "l"(ok ? row + c : row), "r"(ok ? 4 : 0));
            }
        }
    }
    asm volatile("cp.async.commit_group;\n" ::: "memory");
}

// In-place fp32 -> {hi, lo} fp16 pair conversion of one staged buffer (same row split as lm_stage).
__device__ __forceinline__ void lm_convert(const LeafMmaArgs &a, uint32_t *buf) {
    const int TH = a.R + 2;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int rr = warp; rr < kLmParents * TH; rr += kLmThreads / 32) {
        const int pp = rr / TH, tr = rr - pp * TH;     // one division per row
        uint32_t *row = buf + pp * a.ptile + tr * a.TP + 4;
        if (a.vec16) {
            for (int c4 = lane; 4 * c4 < a.W; c4 += 32) {
                uint4 *p = reinterpret_cast<uint4 *>(row + 4 * c4);
                const uint4 v = *p;
                uint2 w01 = lm_split2(__uint_as_float(v.x), __uint_as_float(v.y));
                uint2 w23 = lm_split2(__uint_as_float(v.z), __uint_as_float(v.w));
                *p = make_uint4(w01.x, w01.y, w23.x, w23.y);
            }
        } else {
            for (int c = lane; c < a.W; c += 32) row[c] = lm_split(__uint_as_float(row[c]));
        }
    }
}

// A fragments (hi, lo) of one field from its 4 words (cells e = 0..3 of this lane)
struct Frag { uint32_t h01, h23, l01, l23; };
__device__ __forceinline__ Frag lm_frag(uint32_t w0, uint32_t w1, uint32_t w2, uint32_t w3) {
    return Frag{prmt(w0, w1, 0x5410), prmt(w2, w3, 0x5410), prmt(w0, w1, 0x7632), prmt(w2, w3, 0x7632)};
}

// Warp roles.  Warps w and w + 4 share SM sub-partition w % 4 and TMEM lane quarter w % 4 and
// walk the same chunks; half 0 multiplies the 4 diagonal pairs (g_d, D_d), half 1 the pairs
// (b, g_1), (g_3, g_4), (g_6, -).  Per (thread, class) fp32 totals, TMEM columns
// 256 h + 16 s + i (thread (g, t): parent g, columns a' = 2t, 2t+1; the "sum" slots hold the
// ones column, meaningful on t = 0):
//   half 0, diagonal pair p (d = 0, 2, 5, 7; h_d = g_d + D_d): 3p, 3p+1 = h_d Q'; 3p+2 = sum h_d
//   half 1: 0, 1 = b Q'; 2, 3 = g_1 Q'; 4 = sum b; 5 = sum g_1; 6, 7 = g_3 Q'; 8, 9 = g_4 Q';
//           10 = sum g_3; 11 = sum g_4; 12, 13 = g_6 Q'; 14 = sum g_6
template <int HALF> struct LmRole {
    static constexpr int NP = HALF == 0 ? 4 : 3;          // field pairs
    static constexpr int NV = HALF == 0 ? 12 : 15;        // totals per class
};

template <uint32_t MASK, bool DEV, int HALF>
__device__ __forceinline__ void lm_run(const LeafMmaArgs &a, uint32_t *sm, uint32_t tmem, long long nwork,
                                       long long nsteps) {
    constexpr int NA = mask_count(MASK);
    constexpr int CB = 1 + 8 + 9 * NA;                  // k_hist's class block
    constexpr int NP = LmRole<HALF>::NP, NV = LmRole<HALF>::NV;
    const int warp = threadIdx.x >> 5, q4 = warp & 3, lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
    const uint32_t s0 = (uint32_t)__cvta_generic_to_shared(sm);
    const uint32_t one = g == 0 ? 0x3C003C00u : 0u;     // (1, 1) fp16 in column 0 of the ones tile
    const int TPw = a.TP;
    const long long G = gridDim.x;
    float E[4] = {0.f, 0.f, 0.f, 0.f};                  // sum_y occ(y + d_k) b(y), diagonals (half 0)

    for (long long step = 0; step < nsteps; ++step) {
        const int buf = (int)(step & 1);
        const long long group = blockIdx.x + (step / a.nb) * G;
        const int band = (int)(step % a.nb);
        asm volatile("cp.async.wait_group 0;\n" ::: "memory");
        __syncthreads();
        lm_convert(a, sm + buf * kLmParents * a.ptile);
        __syncthreads();
        if (step + 1 < nsteps) {
            const long long g2 = blockIdx.x + ((step + 1) / a.nb) * G;
            lm_stage(a, s0 + 4u * (uint32_t)((buf ^ 1) * kLmParents * a.ptile), g2, (int)((step + 1) % a.nb), nwork);
        }
        const uint32_t *tw = sm + (buf * kLmParents + g) * a.ptile;   // parent g's tile (words)
        const int ch0 = __ldg(a.wr + band * 5 + q4), ch1 = __ldg(a.wr + band * 5 + q4 + 1);
        if (ch0 < ch1) {
            float run[NV];
#pragma unroll
            for (int i = 0; i < NV; ++i) run[i] = 0.f;
            float c[NP][4], o[NP][4];
#pragma unroll
            for (int p = 0; p < NP; ++p)
#pragma unroll
                for (int i = 0; i < 4; ++i) { c[p][i] = 0.f; o[p][i] = 0.f; }
            // fold the MMA accumulators into the fp32 run (h_d = g_d + D_d combined here)
            auto fold = [&]() {
                if (HALF == 0) {
#pragma unroll
                    for (int p = 0; p < NP; ++p) {
                        run[3 * p] += c[p][0] + c[p][2];
                        run[3 * p + 1] += c[p][1] + c[p][3];
                        run[3 * p + 2] += o[p][0] + o[p][2];
                        E[p] += o[p][2];
                    }
                } else {
#pragma unroll
                    for (int p = 0; p < 2; ++p) {
                        run[6 * p] += c[p][0]; run[6 * p + 1] += c[p][1];
                        run[6 * p + 2] += c[p][2]; run[6 * p + 3] += c[p][3];
                        run[6 * p + 4] += o[p][0]; run[6 * p + 5] += o[p][2];
                    }
                    run[12] += c[2][0]; run[13] += c[2][1]; run[NV - 1] += o[2][0];
                }
#pragma unroll
                for (int p = 0; p < NP; ++p)
#pragma unroll
                    for (int i = 0; i < 4; ++i) { c[p][i] = 0.f; o[p][i] = 0.f; }
            };
            // add the run into the class's TMEM totals
            auto flush = [&](int cls) {
                uint32_t v[16];
                tm_ld16(tmem + 16 * cls, v);
#pragma unroll
                for (int i = 0; i < NV; ++i) {
                    v[i] = __float_as_uint(__uint_as_float(v[i]) + run[i]);
                    run[i] = 0.f;
                }
                tm_st16(tmem + 16 * cls, v);
            };
            // chunk records: a two-deep register ring
            uint4 offA = __ldg(a.offs + (long long)ch0 * 4 + t), qA = __ldg(a.qfr + (long long)ch0 * 32 + lane);
            uint4 dmA = HALF == 0 ? __ldg(a.dmask + (long long)ch0 * 4 + t) : make_uint4(0u, 0u, 0u, 0u);
            const int c1n = ch0 + 1 < ch1 ? ch0 + 1 : ch0;
            uint4 offB = __ldg(a.offs + (long long)c1n * 4 + t), qB = __ldg(a.qfr + (long long)c1n * 32 + lane);
            uint4 dmB = HALF == 0 ? __ldg(a.dmask + (long long)c1n * 4 + t) : make_uint4(0u, 0u, 0u, 0u);
            int cur = (int)(offA.x >> 28), nacc = 0;
            for (int ch = ch0; ch < ch1; ++ch) {
                const uint4 off = offA, q = qA, dm = dmA;
                offA = offB; qA = qB; dmA = dmB;
                const int cn = ch + 2 < ch1 ? ch + 2 : ch1 - 1;
                offB = __ldg(a.offs + (long long)cn * 4 + t);
                qB = __ldg(a.qfr + (long long)cn * 32 + lane);
                if (HALF == 0) dmB = __ldg(a.dmask + (long long)cn * 4 + t);
                const int cls = (int)(off.x >> 28);
                if (cls != cur) {
                    fold();
                    flush(cur);
                    cur = cls;
                    nacc = 0;
                }
                // the 4 cells of this lane in parent g's tile (byte offsets / 4)
                const uint32_t *ce[4] = {tw + ((off.x & 0x0FFFFFFFu) >> 2), tw + (off.y >> 2), tw + (off.z >> 2),
                                         tw + (off.w >> 2)};
                // g_d(y) = b(y - d_k): k = dir_k(d), (dr, dc) = stencil offsets
                auto gfrag = [&](int d) {
                    const int k = d < 4 ? d : d + 1;
                    const int sh = -(k / 3 - 1) * TPw - (k % 3 - 1);
                    return lm_frag(ce[0][sh], ce[1][sh], ce[2][sh], ce[3][sh]);
                };
                const Frag fb = lm_frag(ce[0][0], ce[1][0], ce[2][0], ce[3][0]);
                Frag f0[NP], f1[NP];
                if (HALF == 0) {
                    const uint32_t dmw[4] = {dm.x, dm.y, dm.z, dm.w};
#pragma unroll
                    for (int p = 0; p < 4; ++p) {
                        f0[p] = gfrag(p == 0 ? 0 : p == 1 ? 2 : p == 2 ? 5 : 7);
                        // D_d = occ(y + d_k) b(y): the b fragments under sign-replicated masks
                        const uint32_t m01 = prmt(dmw[p], 0u, 0x9988), m23 = prmt(dmw[p], 0u, 0xBBAA);
                        f1[p] = Frag{fb.h01 & m01, fb.h23 & m23, fb.l01 & m01, fb.l23 & m23};
                    }
                } else {
                    f0[0] = fb;        f1[0] = gfrag(1);
                    f0[1] = gfrag(3);  f1[1] = gfrag(4);
                    f0[2] = gfrag(6);  f1[2] = Frag{0u, 0u, 0u, 0u};
                }
                // three rounds so that dependent MMAs of one accumulator are 2 NP issues apart
#pragma unroll
                for (int p = 0; p < NP; ++p) {
                    lm_mma(c[p], f0[p].h01, f1[p].h01, f0[p].h23, f1[p].h23, q.x, q.y);
                    lm_mma(o[p], f0[p].h01, f1[p].h01, f0[p].h23, f1[p].h23, one, one);
                }
#pragma unroll
                for (int p = 0; p < NP; ++p) {
                    lm_mma(c[p], f0[p].h01, f1[p].h01, f0[p].h23, f1[p].h23, q.z, q.w);
                    lm_mma(o[p], f0[p].l01, f1[p].l01, f0[p].l23, f1[p].l23, one, one);
                }
#pragma unroll
                for (int p = 0; p < NP; ++p) lm_mma(c[p], f0[p].l01, f1[p].l01, f0[p].l23, f1[p].l23, q.x, q.y);
                if (++nacc == kLmFold) {
                    fold();
                    nacc = 0;
                }
            }
            fold();
            flush(cur);
        }
        if (band == a.nb - 1) {
            // epilogue of the group: this warp's totals of parent g into the record of (parent g, quarter)
            const long long wp = group * kLmParents + g;
            const double inv = 1.0 / (double)kLmScale;
            double *rec = a.part + (wp * kLmWarps + q4) * (long long)a.pstride;
            for (int s = 0; s < 16; ++s) {
                uint32_t v[16];
                tm_ld16(tmem + 16 * s, v);
                if (wp < nwork) {
                    double *cb = rec + s * CB;
                    auto val = [&](int i) { return (double)__uint_as_float(v[i]) * inv; };
#pragma unroll
                    for (int i = 0; i < 2; ++i) {
                        const int j = 2 * t + i;
                        if (j < NA) {
                            if (HALF == 0) {
#pragma unroll
                                for (int p = 0; p < 4; ++p) cb[9 + NA + lm_diag_d(p) * NA + j] = val(3 * p + i);
                            } else {
                                cb[9 + j] = val(0 + i);
                                cb[9 + NA + 1 * NA + j] = val(2 + i);
                                cb[9 + NA + 3 * NA + j] = val(6 + i);
                                cb[9 + NA + 4 * NA + j] = val(8 + i);
                                cb[9 + NA + 6 * NA + j] = val(12 + i);
                            }
                        }
                    }
                    if (t == 0) {
                        if (HALF == 0) {
#pragma unroll
                            for (int p = 0; p < 4; ++p) cb[1 + lm_diag_d(p)] = val(3 * p + 2);
                        } else {
                            cb[0] = val(4);
                            cb[1 + 1] = val(5);
                            cb[1 + 3] = val(10);
                            cb[1 + 4] = val(11);
                            cb[1 + 6] = val(14);
                        }
                    }
                }
                uint32_t z[16];
#pragma unroll
                for (int i = 0; i < 16; ++i) z[i] = 0u;
                tm_st16(tmem + 16 * s, z);
            }
            if (HALF == 0 && wp < nwork && t == 0) {
                // E_d = sum_y occ(y + d_k) b(y): diagonals from D_d; orthogonal ones 0 (k_reduce)
#pragma unroll
                for (int d = 0; d < 8; ++d) rec[16 * CB + d] = 0.0;
#pragma unroll
                for (int p = 0; p < 4; ++p) rec[16 * CB + lm_diag_d(p)] = (double)E[p] * inv;
            }
#pragma unroll
            for (int p = 0; p < 4; ++p) E[p] = 0.f;
        }
    }
}

template <uint32_t MASK, bool DEV>
__global__ void __launch_bounds__(kLmThreads, 1) k_leaf_mma(LeafMmaArgs a) {
    static_assert(mask_count(MASK) <= 8, "the (1, Q'_8) tile is not built: |A| = 9 uses the scalar leaf kernel");
    extern __shared__ uint4 lm_smem4[];
    __shared__ uint32_t s_tmem;
    // tiles start after a zeroed 32-word guard: the up-left neighbour of the row-1 col-0 padding
    // cell is word -1 of its tile (the previous tile's zeroed gap, or the guard)
    uint32_t *sm = reinterpret_cast<uint32_t *>(lm_smem4) + kLmGuard;
    if (a.skip && *a.skip) return;
    const long long nwork = DEV ? *a.nwork_dev : a.nwork;
    const long long ngroups = (nwork + kLmParents - 1) / kLmParents;
    if ((long long)blockIdx.x >= ngroups) return;
    const long long nsteps = ((ngroups - blockIdx.x + gridDim.x - 1) / gridDim.x) * a.nb;
    const int warp = threadIdx.x >> 5, half = warp >> 2;

    // per-class totals live in tensor memory: 512 columns x 128 lanes; warps w and w + 4 share
    // lanes 32 (w % 4) .. + 31, half 0 in columns 0..255, half 1 in 256..511
    if (warp == 0) {
        const uint32_t dst = (uint32_t)__cvta_generic_to_shared(&s_tmem);
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(dst));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    // zero the columns the copies never write (tile cols 0..3 and W+4..TP-1 of every row, both
    // buffers), the gaps after the tiles and the guard: halo and padding-cell neighbourhoods
    {
        const int TH = a.R + 2, nz = a.TP - a.W;
        for (int i = threadIdx.x; i < 2 * kLmParents * TH * nz; i += kLmThreads) {
            const int tile = i / (TH * nz), rem = i - tile * (TH * nz);
            const int tr = rem / nz, z = rem - tr * nz;
            const int col = z < 4 ? z : a.W + z;
            sm[tile * a.ptile + tr * a.TP + col] = 0u;
        }
        const int gap = a.ptile - TH * a.TP;             // >= 4 words after every tile
        for (int i = threadIdx.x; i < 2 * kLmParents * gap; i += kLmThreads)
            sm[(i / gap) * a.ptile + TH * a.TP + (i % gap)] = 0u;
        if (threadIdx.x < kLmGuard) sm[(int)threadIdx.x - kLmGuard] = 0u;
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = s_tmem + ((uint32_t)(32 * (warp & 3)) << 16) + 256u * half;
    {
        uint32_t z[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) z[i] = 0u;
        for (int s = 0; s < 16; ++s) tm_st16(tmem + 16 * s, z);
    }
    lm_stage(a, (uint32_t)__cvta_generic_to_shared(sm), blockIdx.x, 0, nwork);
    if (half == 0) lm_run<MASK, DEV, 0>(a, sm, tmem, nwork, nsteps);
    else lm_run<MASK, DEV, 1>(a, sm, tmem, nwork, nsteps);
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(s_tmem));
}

// ---- host: chunk geometry (model-static) and the Q' fragments (after VI / FIB) --------------------
static size_t lm_smem_bytes(const LeafMma &L) {
    return sizeof(uint32_t) * (kLmGuard + 2 * kLmParents * (size_t)L.ptile);
}

qvts_status build_leaf_mma(Model &m) {
    LeafMma &L = m.lm;
    const int H = m.H, W = m.W;
    L.TP = ((W + 6) + 3) & ~3;                        // >= 4 zero columns left, >= 2 right; TP % 4 == 0
    long long budget = 200 * 1024;
    if (const char *ev = std::getenv("QVTS_LM_SMEM")) budget = std::atoll(ev);
    auto ptile_of = [&](int R) { return (((R + 2) * L.TP + 31) & ~31) + 4; };   // = 4 mod 32 words
    int R = H;
    while (R > 1 && (long long)sizeof(uint32_t) * (kLmGuard + 2 * kLmParents * ptile_of(R)) > budget) --R;
    if ((long long)sizeof(uint32_t) * (kLmGuard + 2 * kLmParents * ptile_of(R)) > 227 * 1024) {
        L.nb = 0;                                      // too wide: the scalar leaf kernel is used
        return QVTS_OK;
    }
    L.nb = (H + R - 1) / R;
    L.R = (H + L.nb - 1) / L.nb;
    L.ptile = ptile_of(L.R);
    L.tile_words = (L.R + 2) * L.TP;
    L.h_cs.assign((size_t)L.nb * 17, 0);
    L.h_cells.clear();
    std::vector<uint32_t> offs, dmask;
    std::vector<int32_t> wr;
    const int pad_off[4] = {L.TP + 0, L.TP + 1, L.TP + 2, L.TP + L.TP - 1};   // zero neighbourhoods, residues 0..3
    constexpr int kDiag[4] = {0, 2, 5, 7};          // direction index of the diagonal fields (m8 bit)
    long long nch = 0;
    for (int b = 0; b < L.nb; ++b) {
        const int row0 = b * L.R, nrows = std::min(L.R, H - row0);
        const long long band0 = nch;
        for (int s = 0; s < 16; ++s) {
            L.h_cs[b * 17 + s] = (int)nch;
            std::vector<int> q[4];
            for (int r = row0; r < row0 + nrows; ++r)
                for (int c = 0; c < W; ++c) {
                    const int x = r * W + c;
                    if (!m.occ[x] && m.sig[x] == s) q[c & 3].push_back(x);
                }
            size_t head[4] = {0, 0, 0, 0};
            const int n = (int)(q[0].size() + q[1].size() + q[2].size() + q[3].size());
            const int k = (n + 15) / 16;
            for (int j = 0; j < k; ++j) {
                int cell[16];
                // the 4 positions {e, e+2, e+4, e+6} (e in {0, 1, 8, 9}) are read by lanes t = 0..3 in one
                // shared load: give them distinct tile residues mod 4 where the class allows
                for (int e : {0, 1, 8, 9}) {
                    unsigned used = 0;
                    for (int tt = 0; tt < 4; ++tt) {
                        int best = -1, bestn = 0, anyr = -1, anyn = 0;
                        for (int r = 0; r < 4; ++r) {
                            const int left = (int)(q[r].size() - head[r]);
                            if (left <= 0) continue;
                            if (!(used >> r & 1) && left > bestn) { best = r; bestn = left; }
                            if (left > anyn) { anyr = r; anyn = left; }
                        }
                        if (best < 0) best = anyr;
                        if (best >= 0) {
                            cell[e + 2 * tt] = q[best][head[best]++];
                            used |= 1u << best;
                        } else {
                            int pr = 0;
                            while (pr < 3 && (used >> pr & 1)) ++pr;
                            cell[e + 2 * tt] = -1 - pr;          // padding cell of residue pr
                            used |= 1u << pr;
                        }
                    }
                }
                for (int tt = 0; tt < 4; ++tt) {
                    const int pos[4] = {2 * tt, 2 * tt + 1, 2 * tt + 8, 2 * tt + 9};
                    uint32_t o[4], dm[4] = {0u, 0u, 0u, 0u};
                    for (int e = 0; e < 4; ++e) {
                        const int x = cell[pos[e]];
                        if (x >= 0) {
                            const int r = x / W, c = x % W;
                            o[e] = 4u * (uint32_t)((r - row0 + 1) * L.TP + 4 + c);
                            for (int p = 0; p < 4; ++p)
                                if ((m.m8[x] >> kDiag[p]) & 1) dm[p] |= 0x80u << (8 * e);
                        } else {
                            o[e] = 4u * (uint32_t)pad_off[-1 - x];
                        }
                    }
                    offs.insert(offs.end(), {o[0] | ((uint32_t)s << 28), o[1], o[2], o[3]});
                    dmask.insert(dmask.end(), {dm[0], dm[1], dm[2], dm[3]});
                }
                for (int p = 0; p < 16; ++p) L.h_cells.push_back(cell[p] >= 0 ? cell[p] : -1);
                ++nch;
            }
        }
        L.h_cs[b * 17 + 16] = (int)nch;
        // the band's chunks in 4 equal-count ranges, one per warp (class runs may span warps)
        const long long nb_ch = nch - band0;
        for (int w = 0; w <= kLmWarps; ++w) wr.push_back((int32_t)(band0 + nb_ch * w / kLmWarps));
    }
    L.nchunks = nch;
    QVTS_TRY(upload(L.wr, wr));
    QVTS_TRY(upload(L.offs, offs));
    QVTS_TRY(upload(L.dmask, dmask));
    QVTS_TRY(upload(L.cells, L.h_cells));
    return QVTS_OK;
}

// B fragments per (chunk, lane): column g = a' of Q'(y, a') = src(y, a') - qbar (|A| <= 8), as the
// hi/lo fp16 split of the fp64 value; padding cells and columns g >= |A| are zero.
__global__ void k_leaf_qfrag(const double *__restrict__ src64, const int32_t *__restrict__ cells, long long nchunks,
                             int NA, int HW, double qbar, uint4 *__restrict__ qfr) {
    const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (i >= nchunks * 32) return;
    const long long ch = i >> 5;
    const int lane = (int)(i & 31), g = lane >> 2, t = lane & 3;
    const int pos[4] = {2 * t, 2 * t + 1, 2 * t + 8, 2 * t + 9};
    uint16_t hi[4], lo[4];
    for (int e = 0; e < 4; ++e) {
        const int x = cells[ch * 16 + pos[e]];
        const double v = (x >= 0 && g < NA) ? src64[(size_t)g * HW + x] - qbar : 0.0;
        const __half h = __double2half(v);
        hi[e] = __half_as_ushort(h);
        lo[e] = __half_as_ushort(__double2half(v - (double)__half2float(h)));
    }
    auto pk = [](uint16_t a, uint16_t b) { return (uint32_t)a | ((uint32_t)b << 16); };
    qfr[i] = make_uint4(pk(hi[0], hi[1]), pk(hi[2], hi[3]), pk(lo[0], lo[1]), pk(lo[2], lo[3]));
}

qvts_status build_leaf_qfrag(Model &m, const double *src64, double qbar, bool fib, cudaStream_t st) {
    LeafMma &L = m.lm;
    if (L.nb == 0 || L.nchunks == 0 || m.NA > 8) return QVTS_OK;
    DevBuf &q = fib ? L.qfr_fib : L.qfr;
    QVTS_TRY(q.ensure(sizeof(uint4) * 32 * L.nchunks));
    const long long n = L.nchunks * 32;
    k_leaf_qfrag<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(src64, L.cells.as<int32_t>(), L.nchunks, m.NA, m.HW, qbar,
                                                             q.as<uint4>());
    QVTS_CUDA(cudaGetLastError());
    return QVTS_OK;
}

// Opt-in (QVTS_LEAF_MMA=1, read per call so tests can compare both paths): measured slower than
// the scalar leaf k_hist at C4 (75.7 vs 58.0 ms per plan step), so off by default.
bool leaf_mma_enabled(const Model &m, long long bstride, const float *beliefs) {
    const char *ev = std::getenv("QVTS_LEAF_MMA");
    (void)bstride; (void)beliefs;
    return ev && std::atoi(ev) == 1 && m.lm.nb > 0 && m.lm.nchunks > 0 && m.NA <= 8;
}

template <uint32_t MASK>
static qvts_status launch_leaf_mma_t(Model &m, const float *beliefs, long long bstride, const int32_t *vmap, long long nwork,
                                     int pstride, cudaStream_t st, const int32_t *skip, const long long *nwork_dev) {
    const LeafMma &L = m.lm;
    LeafMmaArgs a;
    a.beliefs = beliefs; a.bstride = bstride; a.vmap = vmap; a.nwork = nwork; a.nwork_dev = nwork_dev; a.skip = skip;
    a.H = m.H; a.W = m.W; a.TP = L.TP; a.R = L.R; a.nb = L.nb; a.ptile = L.ptile;
    a.vec16 = ((m.W & 3) == 0 && (bstride & 3) == 0 && (reinterpret_cast<uintptr_t>(beliefs) & 15) == 0) ? 1 : 0;
    a.wr = L.wr.as<int32_t>(); a.offs = L.offs.as<uint4>(); a.dmask = L.dmask.as<uint4>();
    a.qfr = (m.cur_leaf == QVTS_LEAF_FIB ? L.qfr_fib : L.qfr).as<uint4>();
    a.part = m.part.as<double>(); a.pstride = pstride;
    int dev = 0, nsm = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    const size_t smem = lm_smem_bytes(L);
    auto kfn = nwork_dev ? k_leaf_mma<MASK, true> : k_leaf_mma<MASK, false>;
    QVTS_CUDA(cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    const long long ngroups = (nwork + kLmParents - 1) / kLmParents;
    const unsigned grid = (unsigned)(nwork_dev ? nsm : std::max(1LL, std::min<long long>(nsm, ngroups)));
    kfn<<<grid, kLmThreads, smem, st>>>(a);
    QVTS_CUDA(cudaGetLastError());
    return QVTS_OK;
}

qvts_status launch_leaf_mma(Model &m, const float *beliefs, long long bstride, const int32_t *vmap, long long nwork,
                            int pstride, cudaStream_t st, const int32_t *skip, const long long *nwork_dev) {
    switch (m.mask) {     // |A| <= 8 (A9 keeps the scalar leaf kernel: leaf_mma_enabled)
        case 0x1EF: return launch_leaf_mma_t<0x1EF>(m, beliefs, bstride, vmap, nwork, pstride, st, skip, nwork_dev);
        case 0x0AA: return launch_leaf_mma_t<0x0AA>(m, beliefs, bstride, vmap, nwork, pstride, st, skip, nwork_dev);
        default: break;
    }
    set_error("unsupported action mask for the tensor-core leaf kernel");
    return QVTS_ERR_INVALID_MODEL;
}

int leaf_mma_records() { return kLmWarps; }

}  // namespace qvts
