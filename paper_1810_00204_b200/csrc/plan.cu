// plan.cu — the level-batched QV-tree expansion and its ABI entry points
// qvts_plan_step, qvts_belief_update and the trace accessors.
//
// Per materialised level d (all V-nodes of the level at once; P2 of SURVEY §2.6):
//   k_hist<false>     S1 predict + S2 signature bins of bbar and R(b,a) partials, per (parent, band)
//   k_reduce<false>   S2 fixed-order fp64 reduction -> P(z|b,a), R(b,a); S3 Philox draws, counts
//   k_scan            child offsets (one count read back per level)
//   k_correct         S4 Bayes correction of every unique z, children written with float4 stores
// Leaf level D-1:
//   k_hist<true>      adds S5 bins S_a[sig][a'] = sum bbar_a(y) (Q(y,a') - qbar)
//   k_reduce<true>    leaf values for the sampled z (self-normalised ratio) and Q of the Q-node
// Backup (S6): k_vmax (level D-1), k_backup (levels D-2..0).
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>

#include <cooperative_groups.h>

#include "qvts_internal.cuh"
#include "stencil.cuh"
#include "philox.cuh"

namespace qvts {

// stencil id of the j-th action of MASK for a run-time j: one shift of a packed nibble table
template <uint32_t MASK>
__host__ __device__ constexpr uint64_t action_table() {
    uint64_t t = 0;
    for (int i = 0; i < mask_count(MASK); ++i) t |= (uint64_t)mask_action(MASK, i) << (4 * i);
    return t;
}
template <uint32_t MASK>
__device__ __forceinline__ int action_of(int j) {
    return (int)((action_table<MASK>() >> (4 * j)) & 15u);
}
// laterals of a run-time stencil id (stencil.cuh lat1 / lat2) from packed nibble tables
__host__ __device__ constexpr uint64_t lateral_table(bool second) {
    uint64_t t = 0;
    for (int k = 0; k < 9; ++k) t |= (uint64_t)(second ? lat2(k) : lat1(k)) << (4 * k);
    return t;
}
__device__ __forceinline__ int lat1_rt(int k) { return (int)((lateral_table(false) >> (4 * k)) & 15u); }
__device__ __forceinline__ int lat2_rt(int k) { return (int)((lateral_table(true) >> (4 * k)) & 15u); }

template <uint32_t MASK, bool LEAF>
__host__ __device__ constexpr int hist_cb() {      // class-binned values per thread
    return 1 + 8 + (LEAF ? mask_count(MASK) * 9 : 0);
}
template <uint32_t MASK, bool LEAF>
__host__ __device__ constexpr int hist_nv() { return hist_cb<MASK, LEAF>() + 8; }
constexpr int kRedChunk = 48;                       // values per reduction round

// direction index di (0..7) <-> stencil id k != 4
__host__ __device__ constexpr int dir_k(int di) { return di < 4 ? di : di + 1; }
// orthogonal moves: their target's occupancy is the wall-signature bit (PAPER.md:336 sensors)
__host__ __device__ constexpr bool is_orth(int k) { return k == 1 || k == 3 || k == 5 || k == 7; }
__host__ __device__ constexpr int orth_bit(int k) { return k == 1 ? 0 : k == 3 ? 1 : k == 5 ? 2 : 3; }
// occupancy of y + d_k for every cell of signature class s, or 0 when it is not class-constant
// (the orthogonal ids are exactly the odd ones and orth_bit(k) = k >> 1: no table for a run-time k)
__host__ __device__ constexpr bool orth_is_odd() {
    for (int k = 0; k < 9; ++k)
        if (is_orth(k) != ((k & 1) != 0) || (is_orth(k) && orth_bit(k) != (k >> 1))) return false;
    return true;
}
static_assert(orth_is_odd(), "class_blocked's closed form");
__device__ __forceinline__ double class_blocked(int k, int s) {
    return ((k & 1) && ((s >> (k >> 1)) & 1)) ? 1.0 : 0.0;
}

// ---- S2 tail + S3 (+ S5 tail + S6 leaf backup) ------------------------------------------------
struct ReduceArgs {
    const double *part;
    int pstride, nb;
    long long nwork;
    const int32_t *vmap;
    const float *beliefs;
    long long bstride;
    const uint64_t *vpath;
    const int32_t *vroot;
    const uint32_t *root_step, *root_ep;
    uint32_t seed;
    int level, n;
    const double *O64;
    int ngc;
    const int32_t *gc_cell, *gc_off;   // goal entries grouped by action: [gc_off[j], gc_off[j+1])
    const double *gc_val;
    int goal;
    double p_stay, p_int, p_lat, gamma, qbar;
    double *R, *P;
    uint16_t *cnt, *umask;
    int32_t *U;
    uint8_t *zdraw;
    double *Q, *leafV;
    unsigned long long *counters;   // [0] flagged draws, [1] leaf V-nodes
    // ancestral sampler (NEXT-3): state draws x[q][j] and the tables for x' and z
    const int32_t *xs;
    const uint8_t *m8, *sig;
    int W;
    double acc;
    const int32_t *skip = nullptr;  // device flag: non-zero -> the launch does nothing (best-first)
    const long long *nwork_dev = nullptr;   // device-side parent count (graph-captured plan step)
};

// tree level of a V-node path: one non-zero byte per action level (low nibble a+1 >= 1)
__device__ __forceinline__ int path_level(uint64_t vpath) {
    return vpath ? (64 - __clzll((long long)vpath) + 7) >> 3 : 0;
}

// Alg. 4 steps 2-3 for one sample: x' ~ T(x,a,.) on u2 over the clamped row in stencil order
// (blocked targets merged into the stay entry at first occurrence), then z ~ O(x',.) on u3
// (product over the 4 independent sensors, R7); fp64 CDFs, min{k : u C_last < C_k} (A.5).
__device__ __forceinline__ int ancestral_tail(const ReduceArgs &a, int x, int k, double u2, double u3) {
    int ty[4];
    double tp[4];
    int nt = 0;
    const int m8 = a.m8[x];
    for (int kk = 0; kk < 9; ++kk) {
        double w = 0.0;
        if (k == 4) w = (kk == 4) ? 1.0 : 0.0;
        else if (kk == k) w = a.p_int;
        else if (kk == 4) w = a.p_stay;
        else if (kk == lat1(k) || kk == lat2(k)) w = a.p_lat;
        if (w == 0.0) continue;
        int y = x;
        if (kk != 4 && !((m8 >> nbit(kk)) & 1)) y = x + st_dr(kk) * a.W + st_dc(kk);
        int found = -1;
        for (int e = 0; e < nt; ++e) if (ty[e] == y) found = e;
        if (found >= 0) tp[found] += w;
        else { ty[nt] = y; tp[nt] = w; ++nt; }
    }
    double C[4], acc = 0.0;
    for (int e = 0; e < nt; ++e) { acc += tp[e]; C[e] = acc; }
    double t = u2 * C[nt - 1];
    int xp = ty[nt - 1];
    for (int e = 0; e < nt; ++e) if (t < C[e]) { xp = ty[e]; break; }
    const int sg = a.sig[xp];
    double Cz[16];
    acc = 0.0;
    for (int z = 0; z < 16; ++z) {
        double o = 1.0;
        for (int bb = 0; bb < 4; ++bb) o *= (((z >> bb) & 1) == ((sg >> bb) & 1)) ? a.acc : (1.0 - a.acc);
        acc += o;
        Cz[z] = acc;
    }
    t = u3 * Cz[15];
    for (int z = 0; z < 16; ++z) if (t < Cz[z]) return z;
    return 15;
}

// One CTA per parent V-node, one half-warp per action (Q-node): |A|/2 warps, rounded up.  The CTA
// first brings the parent's record into shared memory (one bulk copy when there is one band, as at
// every leaf level; else the band records summed in fixed band order, fp64); then each half-warp:
// per-action recombination of the linear fields -> M[s], P(z|b,a) (Eq. 3 normaliser), R(b,a)
// (PAPER.md:58), n Philox draws (lane j = sample j), counts; for the leaf level also the Q_MDP value
// of every sampled child, V(z) = qbar + max_a' [sum_s O[s][z] S[s][a']] / P(z), and the Q-node's
// backup Q = R + gamma sum_z (f_z/n) V(z) (Alg. 6 with gamma, R13).
//
// Both sums over signatures, P(z) = sum_s O[s][z] M[s] and the numerators, use that O is the
// Kronecker product of the four sensors' 2x2 matrices K = [[acc, 1-acc], [1-acc, acc]] (PAPER.md:336,
// reading R7): lane s of the half-warp holds the vector, four butterfly stages
// x <- acc x + (1-acc) x(lane ^ 2^b) leave sum_s O[s][z] x[s] on lane z, 4 x 2 shuffles + 2 FP
// operations per vector instead of a 16 x 16 product.
//
// Shared memory (doubles): the parent's record [pstride] | E[8], sum b, 1/n, pad [16] | per action
// [kRedActScratch]: P(z|b,a) [16], the ascending CDF [16], 16 draw counts (ints).
constexpr int kRedActScratch = 16 + 16 + 8;
template <uint32_t MASK>
__host__ __device__ constexpr int reduce_threads() { return (mask_count(MASK) + 1) / 2 * 32; }
template <uint32_t MASK, bool LEAF>
__host__ __device__ constexpr int reduce_smem_doubles(int pstride) {
    return pstride + 16 + mask_count(MASK) * kRedActScratch;
}

// Executed by a CTA of reduce_threads<MASK>() threads for parent w; half-warp h of warp v handles
// action j = 2 v + h.  rsm: reduce_smem_doubles(pstride) doubles of shared memory (16-byte aligned;
// pstride even).
template <uint32_t MASK, bool LEAF, bool ANC>
__device__ void reduce_parent(const ReduceArgs &a, long long w, double *rsm, int nthreads) {
    constexpr int NA = mask_count(MASK);
    constexpr int CB = hist_cb<MASK, LEAF>();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int sl = lane & 15, hf = lane >> 4;  // signature / z / sample of the lane, half-warp
    const unsigned hmask = 0xFFFFu << (16 * hf);   // this half-warp's lanes
    double *sp = rsm;                          // [pstride] band-summed record
    double *sE = rsm + a.pstride;              // [8] blocked-mass totals, [8] = sum b, [9] = 1/n
    const double *pp = a.part + w * a.nb * (long long)a.pstride;
    if (a.nb == 1) {
        // one band: the record is a plain copy -- one bulk (TMA) copy, an mbarrier for completion
        __shared__ alignas(8) unsigned long long s_bar;
        const uint32_t bar = (uint32_t)__cvta_generic_to_shared(&s_bar);
        if (threadIdx.x == 0) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(bar));
            asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
            const uint32_t bytes = (uint32_t)(8 * a.pstride);
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(bar), "r"(bytes) : "memory");
            asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                             (uint32_t)__cvta_generic_to_shared(sp)),
                         "l"(pp), "r"(bytes), "r"(bar)
                         : "memory");
        }
        __syncthreads();                       // the barrier is initialised before anyone waits
        asm volatile(
            "{\n .reg .pred P1;\n WAIT_%=:\n"
            " mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n"
            " @!P1 bra WAIT_%=;\n}\n" ::"r"(bar) : "memory");
    } else {
        // band records summed in fixed band order; a thread takes two adjacent elements per pass
        // as one 16-byte load per band (pstride is even), 4 bands in flight
        const double2 *pp2 = reinterpret_cast<const double2 *>(pp);
        double2 *sp2 = reinterpret_cast<double2 *>(sp);
        const int half = a.pstride >> 1;
        for (int i = threadIdx.x; i < half; i += nthreads) {
            double acc0 = 0.0, acc1 = 0.0;
            for (int bd = 0; bd < a.nb; bd += 4) {
                double2 x[4];
#pragma unroll
                for (int u = 0; u < 4; ++u)
                    if (bd + u < a.nb) x[u] = pp2[(long long)(bd + u) * half + i];
#pragma unroll
                for (int u = 0; u < 4; ++u)
                    if (bd + u < a.nb) { acc0 += x[u].x; acc1 += x[u].y; }
            }
            sp2[i] = make_double2(acc0, acc1);
        }
        __syncthreads();
    }
    // E[d] = sum_y occ(y + d) b(y); orthogonal directions come from the class masses (signature
    // bit: the 8 classes with bit kd/2 set, ascending); thread 8: the belief mass sum_s (class
    // mass), ascending s; thread 9: 1/n; threads 32 + j: action j's stencil ids, packed
    __shared__ uint32_t s_pack[9];
    if (threadIdx.x < 10) {
        const int d = threadIdx.x;
        double e;
        if (d == 9) {
            e = 1.0 / (double)a.n;
        } else if (d == 8) {
            e = 0.0;
#pragma unroll
            for (int s2 = 0; s2 < 16; ++s2) e += sp[s2 * CB];
        } else {
            const int kd = d < 4 ? d : d + 1;
            e = sp[16 * CB + d];
            if (is_orth(kd)) {
                const int bt = kd >> 1;              // orth_bit(kd)
                e = 0.0;
#pragma unroll
                for (int i = 0; i < 8; ++i) {
                    const int s2 = ((i >> bt) << (bt + 1)) | (1 << bt) | (i & ((1 << bt) - 1));
                    e += sp[s2 * CB];
                }
            }
        }
        sE[d] = e;
    } else if (threadIdx.x >= 32 && threadIdx.x < 32 + NA) {
        const int k = action_of<MASK>(threadIdx.x - 32);
        const int k1 = k == 4 ? 4 : lat1_rt(k), k2 = k == 4 ? 4 : lat2_rt(k);
        const int da = k == 4 ? 0 : nbit(k), d1 = k == 4 ? 0 : nbit(k1), d2 = k == 4 ? 0 : nbit(k2);
        s_pack[threadIdx.x - 32] = (uint32_t)(k | k1 << 4 | k2 << 8 | da << 12 | d1 << 16 | d2 << 20);
    }
    __syncthreads();
    const long long v = a.vmap ? (long long)a.vmap[w] : w;
    const float *bp = a.beliefs + v * a.bstride;
    const double mass = sE[8];
    const uint64_t vpath = a.vpath[v];
    const int root = a.vroot[v];
    const uint32_t step = a.root_step[root], ep = a.root_ep[root];
    const double ka = a.acc, kb = 1.0 - a.acc;  // the sensor matrix K
    int nflag = 0, leaves = 0;
    {
    const int jr = 2 * warp + hf;              // this half-warp's action
    const bool act = jr < NA;                  // (odd |A|: the last half-warp only keeps step)
    const int j = act ? jr : NA - 1;
    double *sW = sE + 16 + j * kRedActScratch;
    double *sP = sW;                           // [16] P(z|b,a)
    double *C = sW + 16;                       // [16] ascending CDF
    int *sCnt = reinterpret_cast<int *>(sW + 32);   // [16] draw counts per z
    const long long q = w * NA + j;
    const uint32_t pk = s_pack[j];
    const int k = pk & 15, k1 = (pk >> 4) & 15, k2 = (pk >> 8) & 15;
    const int da = (pk >> 12) & 15, d1 = (pk >> 16) & 15, d2 = (pk >> 20) & 15;
    // the taps' blocked bits for class sl (class_blocked as predicates: h + [blocked] x is the add or h)
    const bool ba = class_blocked(k, sl) != 0.0, b1 = class_blocked(k1, sl) != 0.0, b2 = class_blocked(k2, sl) != 0.0;
    const double *c = sp + sl * CB;            // class sl's record
    // M[s]: bbar_a summed over signature class s (lane s); the counts are cleared
    double Pz;
    {
        const double c0 = c[0];
        double hma = c[1 + da], hm1 = c[1 + d1], hm2 = c[1 + d2];
        if (ba) hma += c0;
        if (b1) hm1 += c0;
        if (b2) hm2 += c0;
        Pz = (k == 4) ? c0 : a.p_stay * c0 + a.p_int * hma + a.p_lat * (hm1 + hm2);
    }
    if (act) sCnt[sl] = 0;
    // P(z|b,a) = sum_s O[s][z] M[s]: the four sensor butterflies, lane z
#pragma unroll
    for (int bt = 1; bt < 16; bt <<= 1) Pz = fma(ka, Pz, kb * __shfl_xor_sync(0xffffffffu, Pz, bt));
    // R(b,a) = (p_stay - 1) sum b - sum c_a b + goal terms, sum c_a b = p_stay mass + p_int E_a + p_lat (E_l1 + E_l2);
    // goal terms G(x, a) b(x): this action's <= 9 entries (model.cu groups them by action), one
    // per lane, tree sum within the half-warp
    double gsum = 0.0;
    if (k != 4) {
        const int g0 = a.gc_off[j], ng = a.gc_off[j + 1] - g0;
        if (sl < ng) gsum = a.gc_val[g0 + sl] * (double)bp[a.gc_cell[g0 + sl]];
    }
#pragma unroll
    for (int o = 8; o > 0; o >>= 1) gsum += __shfl_xor_sync(0xffffffffu, gsum, o);
    double R = 0.0;
    if (sl == 0) {
        if (k == 4) {
            R = -2.0 * mass + 2.0 * (double)bp[a.goal];
        } else {
            const double Rp = a.p_stay * mass + a.p_int * sE[da] + a.p_lat * (sE[d1] + sE[d2]);
            R = (a.p_stay - 1.0) * mass - Rp + gsum;
        }
    }
    if (act) sP[sl] = Pz;
    __syncwarp();
    // ascending-z CDF in fp64, summed sequentially (A.5), on the half-warp's first lane
    if (sl == 0 && act) {
        const double2 *p2 = reinterpret_cast<const double2 *>(sP);
        double2 *c2 = reinterpret_cast<double2 *>(C);
        double acc = 0.0;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            const double2 pv = p2[i];
            double2 cv;
            acc += pv.x;
            cv.x = acc;
            acc += pv.y;
            cv.y = acc;
            c2[i] = cv;
        }
    }
    __syncwarp();
    // S3: n draws keyed by the tree path (Appendix A.2-A.5), lane sl = sample j0 + sl
    const int level = a.level >= 0 ? a.level : path_level(vpath);   // level < 0: from the path
    const uint64_t qpath = vpath | ((uint64_t)(k + 1) << (8 * level));
    if (act) {
        for (int j0 = 0; j0 < a.n; j0 += 16) {
            const int jj = j0 + sl;
            if (jj < a.n) {
                int z;
                const uint4 r = philox4x32_10(make_uint4((uint32_t)jj, (uint32_t)qpath, (uint32_t)(qpath >> 32), step),
                                              make_uint2(a.seed, ep));
                if constexpr (ANC) {   // Alg. 4 literal: x drawn by k_ancestral_x, then x' and z
                    z = ancestral_tail(a, a.xs[q * a.n + jj], k, philox_uniform(r.z), philox_uniform(r.w));
                } else {
                    const double u = philox_uniform(r.x);
                    const double tt = u * C[15];
                    // z = #{k : C_k <= tt} (A.5) by binary search over the non-decreasing CDF; the
                    // gap min_{k<15} |tt - C_k| is attained at the boundaries around tt, C_{z-1} and C_z
                    int lo = 0;
#pragma unroll
                    for (int st = 8; st > 0; st >>= 1)
                        if (C[lo + st - 1] <= tt) lo += st;
                    z = lo + (C[lo] <= tt ? 1 : 0);          // in 0..16
                    double gap = INFINITY;
                    if (z >= 1 && z - 1 < 15) gap = tt - C[z - 1];
                    if (z < 15) gap = fmin(gap, C[z] - tt);
                    z = min(z, 15);
                    nflag += gap < 1e-6 ? 1 : 0;
                }
                if (a.zdraw) a.zdraw[q * a.n + jj] = (uint8_t)z;
                atomicAdd(&sCnt[z], 1);            // integer counts: exact in any order
            }
        }
    }
    __syncwarp();
    const int cntk = act ? sCnt[sl] : 0;       // lane z
    const unsigned um = (__ballot_sync(0xffffffffu, cntk > 0) & hmask) >> (16 * hf);
    const int U = __popc(um);
    if (act) {
        leaves += sl == 0 ? U : 0;
        a.P[q * 16 + sl] = Pz;
        a.cnt[q * 16 + sl] = (uint16_t)cntk;
        if (sl == 0) {
            a.R[q] = R;
            a.umask[q] = (uint16_t)um;
            a.U[q] = U;
        }
    }
    if (LEAF) {
        // S[s][a'] of this action from the linear fields (lane s, every a'), then the same
        // butterflies: lane z holds the numerators sum_s O[s][z] S[s][a']
        double Sv[NA];
#pragma unroll
        for (int j2 = 0; j2 < NA; ++j2) {
            const double zb = c[9 + j2];
            double ha = c[9 + NA + da * NA + j2], h1 = c[9 + NA + d1 * NA + j2], h2 = c[9 + NA + d2 * NA + j2];
            if (ba) ha += zb;
            if (b1) h1 += zb;
            if (b2) h2 += zb;
            Sv[j2] = (k == 4) ? zb : a.p_stay * zb + a.p_int * ha + a.p_lat * (h1 + h2);
        }
#pragma unroll
        for (int bt = 1; bt < 16; bt <<= 1)
#pragma unroll
            for (int j2 = 0; j2 < NA; ++j2) Sv[j2] = fma(ka, Sv[j2], kb * __shfl_xor_sync(0xffffffffu, Sv[j2], bt));
        double best = Sv[0];
#pragma unroll
        for (int j2 = 1; j2 < NA; ++j2) best = fmax(best, Sv[j2]);
        // lane z, z sampled: V(z) = qbar + max_a' num / P(z); the backup sums f_z V(z)
        double fv = 0.0;
        if (cntk > 0) {
            const double Vz = a.qbar + best / Pz;
            if (a.leafV) a.leafV[q * 16 + sl] = Vz;
            fv = (double)cntk * Vz;
        }
#pragma unroll
        for (int o = 8; o > 0; o >>= 1) fv += __shfl_xor_sync(0xffffffffu, fv, o);
        if (sl == 0 && act) a.Q[q] = R + a.gamma * (fv * sE[9]);     // sE[9] = 1/n
    }
    }   // this half-warp's action
    // flagged-draw and leaf counts: per warp, one global atomic each (counts are integers)
    for (int o = 16; o > 0; o >>= 1) {
        nflag += __shfl_xor_sync(0xffffffffu, nflag, o);
        leaves += __shfl_xor_sync(0xffffffffu, leaves, o);
    }
    if (lane == 0 && a.counters) {
        if (nflag) atomicAdd(&a.counters[0], (unsigned long long)nflag);
        if (LEAF && leaves) atomicAdd(&a.counters[1], (unsigned long long)leaves);
    }
    __syncthreads();   // rsm may be reused by the caller
}

// k_reduce: ~1536 resident threads per SM (measured at A8 in round 1: 6 blocks of 256 -> leaf
// launch 7.4 -> 4.5 ms); one half-warp per action
template <uint32_t MASK>
__host__ __device__ constexpr int reduce_min_blocks() {
    return 1536 / reduce_threads<MASK>() > 16 ? 16 : 1536 / reduce_threads<MASK>();
}

// ANC: the ancestral sampler's x' and z tail (a.xs set), compiled apart so the marginal sampler's
// kernel carries none of its registers
template <uint32_t MASK, bool LEAF, bool ANC>
__global__ void __launch_bounds__(reduce_threads<MASK>(), reduce_min_blocks<MASK>()) k_reduce(ReduceArgs a) {
    extern __shared__ double rsm[];
    if (a.skip && *a.skip) return;
    if (a.nwork_dev && (long long)blockIdx.x >= *a.nwork_dev) return;
    reduce_parent<MASK, LEAF, ANC>(a, blockIdx.x, rsm, reduce_threads<MASK>());
}

// ---- NEXT-3: the state draw x ~ b of Alg. 4 for every sample of every Q-node of a parent ------
// One CTA per parent: fp64 sums of 256-cell chunks (warp per chunk, fixed order), their exclusive
// prefix, then per (action, sample) target t = u1 * C_total: the chunk by binary search and the
// cell by a sequential fp64 scan inside it, min{x : t < C_x} (A.5; zero-mass cells never drawn).
// chunk of the two-level prefix: a multiple of 32 cells, at most 2048 chunks (32 KB of shared
// prefix for any map)
__host__ __device__ constexpr int ancestral_chunk(int HW) {
    return ((HW + 2047) / 2048 + 31) / 32 * 32 < 32 ? 32 : ((HW + 2047) / 2048 + 31) / 32 * 32;
}
__host__ __device__ constexpr int ancestral_nch(int HW) { return (HW + ancestral_chunk(HW) - 1) / ancestral_chunk(HW); }

template <uint32_t MASK>
__global__ void __launch_bounds__(256) k_ancestral_x(const float *__restrict__ beliefs, long long bstride,
                                                     const int32_t *vmap, long long nwork, int HW,
                                                     const uint64_t *vpath, const int32_t *vroot,
                                                     const uint32_t *root_step, const uint32_t *root_ep,
                                                     uint32_t seed, int level, int n, int32_t *xs,
                                                     const int32_t *skip = nullptr,
                                                     const long long *nwork_dev = nullptr) {
    constexpr int NA = mask_count(MASK);
    extern __shared__ double sx[];   // [nch] chunk sums, [nch + 1] exclusive prefix
    __shared__ double s_wtot[8];
    if (skip && *skip) return;
    if (nwork_dev && (long long)blockIdx.x >= *nwork_dev) return;   // graph path: worst-case grid
    const long long w = blockIdx.x;
    const long long v = vmap ? (long long)vmap[w] : w;
    const float *__restrict__ b = beliefs + v * bstride;
    const int CH = ancestral_chunk(HW), nch = ancestral_nch(HW);
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
    double *csum = sx, *cpre = sx + nch;
    // fp64 chunk sums: a warp reads 128 consecutive cells per pass (4 per lane), each lane sums
    // its 4 in order, 8-lane butterflies give the 32-cell sums, and a chunk of CH cells adds its
    // CH / 32 pieces in order (lane 0 of each 8-lane group)
    const bool v4 = ((HW & 3) == 0) && ((reinterpret_cast<uintptr_t>(b) & 15) == 0);
    if (CH == 32) {   // four chunks per 128-cell pass (maps up to 64K cells), 4 passes in flight
        const int nblk = (nch + 3) / 4;
        for (int blk0 = warp; blk0 < nblk; blk0 += 32) {
            float4 f[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int x = 128 * (blk0 + 8 * u) + 4 * lane;
                f[u] = make_float4(0.f, 0.f, 0.f, 0.f);
                if (blk0 + 8 * u < nblk) {
                    if (v4 && x + 3 < HW) {
                        f[u] = __ldg(reinterpret_cast<const float4 *>(b + x));
                    } else {
                        if (x < HW) f[u].x = __ldg(b + x);
                        if (x + 1 < HW) f[u].y = __ldg(b + x + 1);
                        if (x + 2 < HW) f[u].z = __ldg(b + x + 2);
                        if (x + 3 < HW) f[u].w = __ldg(b + x + 3);
                    }
                }
            }
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int blk = blk0 + 8 * u;
                double q = (((double)f[u].x + (double)f[u].y) + (double)f[u].z) + (double)f[u].w;
#pragma unroll
                for (int o = 1; o < 8; o <<= 1) q += __shfl_xor_sync(0xffffffffu, q, o);
                if (blk < nblk && (lane & 7) == 0 && 4 * blk + (lane >> 3) < nch) csum[4 * blk + (lane >> 3)] = q;
            }
        }
    } else for (int c = warp; c < nch; c += 8) {
        double s = 0.0;
        for (int p0 = c * CH; p0 < min(HW, (c + 1) * CH); p0 += 128) {
            const int x = p0 + 4 * lane;
            double q = 0.0;
#pragma unroll
            for (int i = 0; i < 4; ++i)
                if (x + i < HW && x + i < (c + 1) * CH) q += (double)__ldg(b + x + i);
#pragma unroll
            for (int o = 1; o < 8; o <<= 1) q += __shfl_xor_sync(0xffffffffu, q, o);
            // pieces of this pass: lanes 0, 8, 16, 24 hold the 32-cell sums, in cell order
#pragma unroll
            for (int g = 0; g < 4; ++g) s += __shfl_sync(0xffffffffu, q, 8 * g);
        }
        if (lane == 0) csum[c] = s;
    }
    __syncthreads();
    // exclusive prefix over the chunks in a fixed order: each thread a run of consecutive chunks,
    // the run totals scanned across the CTA (warp shuffles, then the 8 warp totals in order)
    const int per = (nch + 255) / 256, c0 = t * per, c1 = min(nch, c0 + per);
    double run = 0.0;
    for (int c = c0; c < c1; ++c) run += csum[c];
    double inc = run;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const double y = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += y;
    }
    if (lane == 31) s_wtot[warp] = inc;
    __syncthreads();
    double base = 0.0;
    for (int w2 = 0; w2 < warp; ++w2) base += s_wtot[w2];
    double acc0 = base + (inc - run);         // exclusive prefix of this thread's run
    for (int c = c0; c < c1; ++c) { cpre[c] = acc0; acc0 += csum[c]; }
    if (t == 255) {
        double tot = 0.0;
        for (int w2 = 0; w2 < 8; ++w2) tot += s_wtot[w2];
        cpre[nch] = tot;
    }
    __syncthreads();
    const double total = cpre[nch];
    const uint64_t vp = vpath[v];
    if (level < 0) level = path_level(vp);
    const int root = vroot[v];
    const uint32_t step = root_step[root], ep = root_ep[root];
    for (int idx = t; idx < NA * n; idx += 256) {
        const int j = idx / n, s = idx % n;
        int kk = 0;
#pragma unroll
        for (int i = 0; i < NA; ++i) if (i == j) kk = mask_action(MASK, i);
        const uint64_t qpath = vp | ((uint64_t)(kk + 1) << (8 * level));
        const uint4 r = philox4x32_10(make_uint4((uint32_t)s, (uint32_t)qpath, (uint32_t)(qpath >> 32), step),
                                      make_uint2(seed, ep));
        const double tt = philox_uniform(r.y) * total;
        int lo = 0, hi = nch - 1;                   // first chunk whose end exceeds tt
        while (lo < hi) {
            const int mid = (lo + hi) >> 1;
            if (tt < cpre[mid + 1]) hi = mid; else lo = mid + 1;
        }
        double acc = cpre[lo];
        int xsel = -1, last = -1;
        const int x1 = min(HW, (lo + 1) * CH);
        for (int x = lo * CH; x < x1; ++x) {
            const double bv = (double)__ldg(b + x);
            acc += bv;
            if (bv > 0.0) last = x;
            if (tt < acc) { xsel = x; break; }
        }
        // rounding at the very end of a chunk (the prefix and this scan sum in different orders)
        if (xsel < 0) xsel = last >= 0 ? last : lo * CH;
        xs[((long long)w * NA + j) * n + s] = xsel;
    }
}

// ---- S1 + S2 (+ S5): signature-binned histograms ----------------------------------------------
// Linear form of the clamped predict: with the 8 clamped source fields
//   h_k(y) = b(y - d_k) + occ(y + d_k) b(y)          (k = the 8 moving stencil directions)
// every action's prediction is bbar_a = p_stay b + p_int h_a + p_lat (h_l1 + h_l2) (stay: b).
// Everything the Q-node needs is linear in bbar, so the kernel accumulates per wall-signature
// class s (the observation class of O(y,z)) only
//   mass_s = sum b,  HM_s[k] = sum h_k,  and for leaves Zb_s[a'] = sum b Q'(.,a'),
//   H_s[k][a'] = sum h_k Q'(.,a')   (Q' = Q - qbar, SURVEY c.6 rule 5)
// plus E[k] = sum occ(y + d_k) b(y) for R(b,a); k_reduce recombines them per action in fp64.
// One CTA = 2 parents x one row band: 256 threads = 128 slot-threads x 2 parents, the parents in
// the two half-warps so the static per-slot loads (entry, Q') are shared; one fp64 partial per
// (parent, band).  The plan's leaf level runs leaf.cu's k_leaf instead (same values, class-fixed
// slots across bands, packed parent pairs) for the action sets it covers.

// ---- S4: Bayes correction of every unique z of a Q-node ----------------------------------------
// One CTA = one Q-node x 1024 cells (4 consecutive cells of one row per thread).  The thread
// predicts bbar_a for its 4 cells once (linear form of k_hist) and writes every child
// b'_z = O(y,z) bbar_a(y) / P(z|b,a) (Eq. 3) with float4 stores; w_z[s] = O[s][z] / P(z) is
// formed in fp64 and staged in shared memory.
struct CorrectArgs {
    const float *beliefs;
    long long bstride;
    const int32_t *vmap;
    const uint8_t *m8, *cell;
    const double *O64;
    const double *P;
    const uint16_t *cnt, *umask;
    const int32_t *off;
    const uint64_t *vpath;
    const int32_t *vroot;
    int level;
    float *child;
    long long cstride;
    uint64_t *cpath;
    int32_t *cparent, *cz, *cf, *croot;
    int H, W, G, ntiles, rows_cta;
    float p_int, p_stay, p_lat;
    long long qsel;   // >= 0: only this Q-node (belief_update)
    const int32_t *sel_q, *sel_z, *sel_out;   // optional per-block-group selection (episodes)
    const int32_t *skip = nullptr;             // device flag (best-first)
    const long long *cbase_dev = nullptr;      // device child-index base (best-first pool)
    const long long *nwork_dev = nullptr;      // device-side parent count (graph-captured plan step)
    long long q0 = 0;                          // first Q-node of this launch (chunked launches)
    int stage_tp = 0;                          // > 0: the CTA's parent rows (+ halo) are staged in shared
                                               // memory with this row pitch (correct_stage)
    int vec_in = 0, vec_out = 0;               // 16-byte row access to the parents / children: W, the
                                               // strides AND the base pointers allow it (correct_stage)
};

// bbar_a for 4 consecutive cells (r, c0..c0+3): bbar = p_stay b + p_int h_a + p_lat (h_l1 + h_l2),
// h_k = b(y - d_k) + occ(y + d_k) b(y); stay: bbar = b.  nbh holds rows r-1..r+1, cols c0-1..c0+4.
template <int K>
__device__ __forceinline__ void correct_predict(const CorrectArgs &a, int r, int c0, const float (&nbh)[3][6],
                                                float (&bb)[4], int (&sg)[4]) {
#pragma unroll
    // cell info of the 4 cells in one 32-bit load each when the row is 4-aligned
    const int x0 = r * a.W + c0;
    uint32_t info4 = 0, m84 = 0;
    const bool al = ((a.W & 3) == 0) && (c0 + 3 < a.W);
    if (al) {
        info4 = __ldg(reinterpret_cast<const unsigned int *>(a.cell + x0));
        if (K != 4) m84 = __ldg(reinterpret_cast<const unsigned int *>(a.m8 + x0));
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int c = c0 + i;
        bb[i] = 0.f;
        sg[i] = 0;
        if (c >= a.W) continue;
        const int x = x0 + i;
        const int info = al ? (int)((info4 >> (8 * i)) & 0xFFu) : (int)__ldg(a.cell + x);
        sg[i] = info & 15;
        if (info & 16) continue;                      // occupied: no mass
        const float b0 = nbh[1][1 + i];
        if (K == 4) {
            bb[i] = b0;
        } else {
            const int m8 = al ? (int)((m84 >> (8 * i)) & 0xFFu) : (int)__ldg(a.m8 + x);
            constexpr int L1 = lat1(K), L2 = lat2(K);
            const float sa = nbh[1 - st_dr(K)][1 + i - st_dc(K)];
            const float s1 = nbh[1 - st_dr(L1)][1 + i - st_dc(L1)];
            const float s2 = nbh[1 - st_dr(L2)][1 + i - st_dc(L2)];
            const float ha = ((m8 >> nbit(K)) & 1) ? sa + b0 : sa;
            const float h1 = ((m8 >> nbit(L1)) & 1) ? s1 + b0 : s1;
            const float h2 = ((m8 >> nbit(L2)) & 1) ? s2 + b0 : s2;
            bb[i] = fmaf(a.p_lat, h1 + h2, fmaf(a.p_int, ha, a.p_stay * b0));
        }
    }
}

struct HistArgs {
    const float *beliefs;
    long long bstride;
    const int32_t *vmap;
    long long nwork;
    const BandInfo *bands;
    int nb;
    const uint32_t *entries;
    const float4 *qlist;
    int H, W, TW, tstride, red_off, sums_off;
    int vec16;            // 16-byte cp.async staging (W % 4 == 0, 16-byte aligned rows)
    double *part;
    int pstride;
    const int32_t *skip = nullptr;  // device flag (best-first)
    const long long *nwork_dev = nullptr;   // device-side parent count (graph-captured plan step)
    unsigned long long *skipped = nullptr;  // (CTA, band) tiles skipped (active-tile skipping)
};

template <uint32_t MASK, bool LEAF, bool DEV = false>
__global__ void __launch_bounds__(kPairThreads, 2) k_hist(HistArgs a) {
    constexpr int NA = mask_count(MASK);
    constexpr int NAP = (NA + 3) & ~3;
    constexpr int CB = hist_cb<MASK, LEAF>();
    constexpr int NV = hist_nv<MASK, LEAF>();
    constexpr int NOUT = 16 * CB + 8;
    constexpr int T = kHistThreads;
    constexpr int ZB = 9, HQ = 9 + NA;               // offsets in the flat accumulator array
    extern __shared__ float4 smem4[];
    if (a.skip && *a.skip) return;
    float *smem = reinterpret_cast<float *>(smem4);
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
    const int p = lane >> 4;                       // parent of this half-warp
    const int st = warp * 16 + (lane & 15);        // slot-thread 0..T-1
    const int band = blockIdx.x % a.nb;
    const long long pair = blockIdx.x / a.nb;
    // DEV (graph-captured step): the parent count lives on the device and the grid is worst-case
    const long long nwork = DEV ? *a.nwork_dev : a.nwork;
    if (DEV && 2 * pair >= nwork) return;
    const BandInfo *bi = a.bands + band;
    const int row0 = bi->row0, nrows = bi->nrows, L = bi->L;
    const long long soff = bi->slot_off;
    const int TH = nrows + 2;

    // stage both parents' bands (+ zero halo) with cp.async; rows off the map and a missing
    // second parent are zero-filled by the copy itself (src-size 0)
    const int TP = a.TW;                              // tile row pitch; column c sits at c + 4
#pragma unroll
    for (int pp = 0; pp < 2; ++pp) {
        const long long wp = 2 * pair + pp;
        const bool vp = wp < nwork;
        const long long vv = vp ? (a.vmap ? (long long)a.vmap[wp] : wp) : 0;
        const float *__restrict__ b = a.beliefs + vv * a.bstride;
        float *tile = smem + pp * a.tstride;
        const uint32_t sbase = (uint32_t)__cvta_generic_to_shared(tile);
        if (a.vec16) {
            // warp per tile row, lanes over the row's 16-byte groups (no index division)
            const int W4 = a.W >> 2;
            for (int tr = warp; tr < TH; tr += kPairThreads / 32) {
                const int r = row0 - 1 + tr;
                const bool ok = vp && r >= 0 && r < a.H;
                const float *src = ok ? b + (long long)r * a.W : b;
                const uint32_t dst = sbase + 4u * (uint32_t)(tr * TP + 4);
                for (int c4 = lane; c4 < W4; c4 += 32)
                    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(dst + 16u * c4),
                                 "l"(ok ? src + 4 * c4 : src), "r"(ok ? 16 : 0));
            }
        } else {
            for (int tr = warp; tr < TH; tr += kPairThreads / 32) {
                const int r = row0 - 1 + tr;
                const bool ok = vp && r >= 0 && r < a.H;
                const float *src = ok ? b + (long long)r * a.W : b;
                const uint32_t dst = sbase + 4u * (uint32_t)(tr * TP + 4);
                for (int c = lane; c < a.W; c += 32)
                    asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;\n" ::"r"(dst + 4u * c),
                                 "l"(ok ? src + c : src), "r"(ok ? 4 : 0));
            }
        }
        // halo columns, and the row padding the copies never write: the skip scan below reads
        // whole rows, so stale shared memory there would decide skips at random
        for (int i = t; i < TH * (TP - a.W); i += kPairThreads) {
            const int tr = i / (TP - a.W), j = i - tr * (TP - a.W);
            tile[tr * TP + (j < 4 ? j : a.W + j)] = 0.f;
        }
        for (int i = t; i < 3 * TP; i += kPairThreads) tile[TH * TP + i] = 0.f;   // zero rows: pad cell
    }
    asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;\n" ::: "memory");
    __syncthreads();
    // Active-tile skipping: when both parents' bands (with halo) hold no
    // belief mass, every accumulated value is exactly zero -- write zero partials, skip the work.
    {
        int any = 0;
        for (int pp = 0; pp < 2; ++pp) {
            const float4 *t4 = reinterpret_cast<const float4 *>(smem + pp * a.tstride);
            for (int i = t; i < (TH * TP) / 4; i += kPairThreads) {
                const float4 v = t4[i];
                any |= (v.x != 0.f) | (v.y != 0.f) | (v.z != 0.f) | (v.w != 0.f);
            }
        }
        if (!__syncthreads_or(any)) {
            constexpr int NOUT0 = 16 * CB + 8;
            for (int o = t; o < 2 * NOUT0; o += kPairThreads) {
                const int pp = o / NOUT0, oo = o % NOUT0;
                const long long wp = 2 * pair + pp;
                if (wp < nwork) a.part[(wp * a.nb + band) * (long long)a.pstride + oo] = 0.0;
            }
            if (t == 0 && a.skipped) atomicAdd(a.skipped, 1ULL);
            return;
        }
    }
    const float *tile = smem + p * a.tstride;

    float acc[NV];
#pragma unroll
    for (int i = 0; i < NV; ++i) acc[i] = 0.f;
    // one cell of the slot stream: 32-bit shared addresses, neighbours at immediate offsets from
    // the cell and from the rows above / below.  Padding slots point at a cell of the zero rows
    // after the tile (m8 = 0, Q' = 0), so they need no branch.
    const uint32_t tbase = (uint32_t)__cvta_generic_to_shared(smem + p * a.tstride);
    const uint32_t TP4 = 4u * (uint32_t)TP;
    auto load_nb = [&](uint32_t e, float (&nb)[9]) {
        const uint32_t c0 = tbase + ((e & 0xFFFFu) << 2);
        const uint32_t cu = c0 - TP4, cd = c0 + TP4;
        asm volatile("ld.shared.f32 %0, [%1+-4];" : "=f"(nb[0]) : "r"(cu));
        asm volatile("ld.shared.f32 %0, [%1];" : "=f"(nb[1]) : "r"(cu));
        asm volatile("ld.shared.f32 %0, [%1+4];" : "=f"(nb[2]) : "r"(cu));
        asm volatile("ld.shared.f32 %0, [%1+-4];" : "=f"(nb[3]) : "r"(c0));
        asm volatile("ld.shared.f32 %0, [%1];" : "=f"(nb[4]) : "r"(c0));
        asm volatile("ld.shared.f32 %0, [%1+4];" : "=f"(nb[5]) : "r"(c0));
        asm volatile("ld.shared.f32 %0, [%1+-4];" : "=f"(nb[6]) : "r"(cd));
        asm volatile("ld.shared.f32 %0, [%1];" : "=f"(nb[7]) : "r"(cd));
        asm volatile("ld.shared.f32 %0, [%1+4];" : "=f"(nb[8]) : "r"(cd));
    };
    auto cell = [&](uint32_t e, const float (&nb)[9], const float4 (&qv)[LEAF ? NAP / 4 : 1]) {
        const uint32_t m8 = e >> 16;
        float q[LEAF ? NAP : 1];
        if (LEAF) {
#pragma unroll
            for (int h = 0; h < (LEAF ? NAP / 4 : 0); ++h) {
                q[4 * h] = qv[h].x; q[4 * h + 1] = qv[h].y; q[4 * h + 2] = qv[h].z; q[4 * h + 3] = qv[h].w;
            }
        }
        const float b0 = nb[4];
        acc[0] += b0;
        if (LEAF) {
#pragma unroll
            for (int j = 0; j < (LEAF ? NA : 0); ++j) acc[ZB + j] = fmaf(b0, q[j], acc[ZB + j]);
        }
#pragma unroll
        for (int d = 0; d < 8; ++d) {
            const int k = dir_k(d);
            float h = nb[8 - k];
            // blocked target: the mass stays at y.  For the 4 orthogonal directions occupancy is a
            // bit of the cell's wall signature, i.e. constant over the class: k_reduce adds it.
            if (!is_orth(k) && (m8 & (1u << d))) {
                h += b0;
                acc[CB + d] += b0;
            }
            acc[1 + d] += h;
            if (LEAF) {
#pragma unroll
                for (int j = 0; j < (LEAF ? NA : 0); ++j) acc[HQ + d * NA + j] = fmaf(h, q[j], acc[HQ + d * NA + j]);
            }
        }
    };
    // Slot streams are padded on the host by >= 4 steps (pads = the zero cell), so the loads
    // below never need a bound check.  Entries run two slots ahead, Q' rows one (ping-pong), the
    // next cell's neighbourhood is loaded before the current cell is accumulated.
    const uint32_t *ep = a.entries + soff + st;
    const float4 *qp = a.qlist + (soff + st) * (NAP / 4);
    constexpr int QSTEP = T * (NAP / 4);
    uint32_t eA = __ldg(ep), eB = __ldg(ep + T), eC, eD;
    float4 qA[LEAF ? NAP / 4 : 1], qB[LEAF ? NAP / 4 : 1];
    if (LEAF) {
#pragma unroll
        for (int h = 0; h < (LEAF ? NAP / 4 : 0); ++h) qA[h] = __ldg(qp + h);
    }
    float nbA[9], nbB[9];
    load_nb(eA, nbA);
    for (int i = 0; i < L; i += 2) {
        eC = __ldg(ep + 2 * T);
        if (LEAF) {
#pragma unroll
            for (int h = 0; h < (LEAF ? NAP / 4 : 0); ++h) qB[h] = __ldg(qp + QSTEP + h);
        }
        load_nb(eB, nbB);
        cell(eA, nbA, qA);
        eD = __ldg(ep + 3 * T);
        if (LEAF) {
#pragma unroll
            for (int h = 0; h < (LEAF ? NAP / 4 : 0); ++h) qA[h] = __ldg(qp + 2 * QSTEP + h);
        }
        load_nb(eC, nbA);
        cell(eB, nbB, qB);
        eA = eC;
        eB = eD;
        ep += 2 * T;
        qp += 2 * QSTEP;
    }
    __syncthreads();   // tiles are dead; reuse the region for the fixed-order class reduction
    constexpr int RS = T + 1;
    float *red = smem + a.red_off;                   // [2][kRedChunk][RS]
    double *sums = reinterpret_cast<double *>(smem + a.sums_off);   // [2][NOUT]
#pragma unroll
    for (int c0 = 0; c0 < NV; c0 += kRedChunk) {
#pragma unroll
        for (int i = 0; i < kRedChunk; ++i)
            if (c0 + i < NV) red[(p * kRedChunk + i) * RS + st] = acc[c0 + i];
        __syncthreads();
        // outputs of this chunk: (class, parent, value) with the class varying slowest, so each
        // thread's outputs fall in different classes (class 0 holds ~40% of the slot-threads);
        // every sum runs in a fixed order over 4 interleaved fp64 accumulators.
        const int nvals = (NV - c0 < kRedChunk) ? NV - c0 : kRedChunk;
        for (int o = t; o < 17 * 2 * nvals; o += kPairThreads) {
            const int cls = o / (2 * nvals), r = o % (2 * nvals);
            const int pp = r / nvals, vi = r % nvals, vv = c0 + vi;
            const float *rp = red + (pp * kRedChunk + vi) * RS;
            int t0, t1;
            if (cls < 16) {
                if (vv >= CB) continue;
                t0 = bi->cs[cls];
                t1 = bi->cs[cls + 1];
            } else {
                if (vv < CB) continue;
                t0 = 0;
                t1 = T;
            }
            double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
            int th = t0;
            for (; th + 3 < t1; th += 4) {
                s0 += (double)rp[th];
                s1 += (double)rp[th + 1];
                s2 += (double)rp[th + 2];
                s3 += (double)rp[th + 3];
            }
            for (; th < t1; ++th) s0 += (double)rp[th];
            const double sm = (s0 + s1) + (s2 + s3);
            if (cls < 16) sums[pp * NOUT + cls * CB + vv] = sm;
            else sums[pp * NOUT + 16 * CB + (vv - CB)] = sm;
        }
        __syncthreads();
    }
    for (int o = t; o < 2 * NOUT; o += kPairThreads) {
        const int pp = o / NOUT, oo = o % NOUT;
        const long long wp = 2 * pair + pp;
        if (wp < nwork) a.part[(wp * a.nb + band) * (long long)a.pstride + oo] = sums[o];
    }
}

// ---- child offsets: single-CTA exclusive scan -------------------------------------------------
__global__ void __launch_bounds__(1024) k_scan(const int32_t *__restrict__ U, int32_t *__restrict__ off, long long n,
                                               long long *total, const int32_t *skip = nullptr,
                                               const long long *nwork_dev = nullptr, int na = 1) {
    __shared__ long long wsum[32];
    __shared__ long long carry_s;
    if (skip && *skip) return;
    if (nwork_dev) n = *nwork_dev * na;                // Q-nodes of the level, from the device count
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
    if (t == 0) carry_s = 0;
    __syncthreads();
    for (long long base = 0; base < n; base += 1024) {
        const long long i = base + t;
        const long long x = i < n ? U[i] : 0;
        long long s = x;
        for (int o = 1; o < 32; o <<= 1) {
            const long long y = __shfl_up_sync(0xffffffffu, s, o);
            if (lane >= o) s += y;
        }
        if (lane == 31) wsum[warp] = s;
        __syncthreads();
        if (warp == 0) {
            long long ws = wsum[lane];
            for (int o = 1; o < 32; o <<= 1) {
                const long long y = __shfl_up_sync(0xffffffffu, ws, o);
                if (lane >= o) ws += y;
            }
            wsum[lane] = ws;
        }
        __syncthreads();
        const long long carry = carry_s;
        const long long excl = carry + (warp ? wsum[warp - 1] : 0) + s - x;
        if (i < n) off[i] = (int32_t)excl;
        __syncthreads();
        if (t == 1023) carry_s = carry + wsum[31];
        __syncthreads();
    }
    if (t == 0) *total = carry_s;
}

template <uint32_t MASK>
__global__ void __launch_bounds__(256) k_correct(CorrectArgs a) {
    constexpr int NA = mask_count(MASK);
    if (a.skip && *a.skip) return;
    const long long grp = blockIdx.x / a.ntiles;
    if (a.nwork_dev && !a.sel_q && grp >= *a.nwork_dev * NA) return;
    const long long q = a.sel_q ? (long long)a.sel_q[grp] : (a.qsel >= 0 ? a.qsel : a.q0 + grp);
    const int tile = blockIdx.x % a.ntiles;
    const long long w = q / NA;
    const int j = (int)(q % NA);
    const int k = action_of<MASK>(j);
    const long long v = a.vmap ? (long long)a.vmap[w] : w;
    const unsigned um = a.sel_q ? (1u << a.sel_z[grp]) : a.umask[q];
    const int U = __popc(um);
    const long long base = (a.sel_q ? (long long)a.sel_out[grp] : (a.qsel >= 0 ? 0 : a.off[q])) +
                           (a.cbase_dev ? *a.cbase_dev : 0);
    // [signature s][rank u] = O[s][z_u] / P(z_u); row pitch 18 so the 16 rows sit in distinct
    // bank pairs and a cell reads two children's weights with one 8-byte load
    __shared__ __align__(16) float s_w[16][18];
    {
        const int t = threadIdx.x;
        const int u = t >> 4, sg = t & 15;
        if (u < U) {
            unsigned rem = um;
            for (int i = 0; i < u; ++i) rem &= rem - 1;
            const int z = __ffs(rem) - 1;
            // a zero-likelihood z (only reachable through the belief_update ABI, which then reports
            // QVTS_ERR_ZERO_LIKELIHOOD) writes zeros instead of O/0 = inf/NaN
            const double pz = a.P[q * 16 + z];
            s_w[sg][u] = pz > 1e-30 ? (float)(a.O64[sg * 16 + z] / pz) : 0.f;
            if (tile == 0 && sg == 0 && a.cpath) {
                const long long c = base + u;
                const int level = a.level >= 0 ? a.level : path_level(a.vpath[v]);
                a.cpath[c] = a.vpath[v] | ((uint64_t)(k + 1) << (8 * level)) | ((uint64_t)z << (8 * level + 4));
                a.cparent[c] = (int32_t)q;
                a.cz[c] = z;
                a.cf[c] = a.cnt[q * 16 + z];
                a.croot[c] = a.vroot[v];
            }
        }
    }
    // this CTA covers rows [tile * rows_cta, +rows_cta): 4 consecutive cells per thread, rows_it
    // rows per pass
    const int W = a.W;
    const float *__restrict__ b = a.beliefs + v * a.bstride;
    const bool vec = a.vec_in != 0;
    const int r_end = min(a.H, (tile + 1) * a.rows_cta);
    // staged path: the parent's rows [r0 - 1, r_end + 1) land in shared memory in one cp.async
    // burst (row pitch stage_tp, column c at c + 4, zero halo columns and off-map rows), so the
    // neighbourhood loads below no longer wait on L2 one pass at a time
    extern __shared__ float4 c_smem4[];
    float *stile = reinterpret_cast<float *>(c_smem4);
    const int r0 = tile * a.rows_cta;
    if (a.stage_tp > 0) {
        const int TPc = a.stage_tp, nr = r_end - r0 + 2, W4 = W >> 2;
        const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
        for (int tr = warp; tr < nr; tr += 8) {
            const int rr = r0 - 1 + tr;
            const bool ok = rr >= 0 && rr < a.H;
            const float *src = ok ? b + (long long)rr * W : b;
            const uint32_t dst = (uint32_t)__cvta_generic_to_shared(stile + tr * TPc + 4);
            for (int c4 = lane; c4 < W4; c4 += 32)
                asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(dst + 16u * c4),
                             "l"(ok ? src + 4 * c4 : src), "r"(ok ? 16 : 0));
            if (lane == 0) {
                stile[tr * TPc + 3] = 0.f;
                stile[tr * TPc + 4 + W] = 0.f;
            }
        }
        asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;\n" ::: "memory");
    }
    __syncthreads();
    for (int idx = threadIdx.x; idx < a.rows_cta * a.G; idx += 256) {
        const int r = tile * a.rows_cta + idx / a.G, c0 = 4 * (idx % a.G);
        if (r >= r_end) break;
        // rows r-1..r+1, columns c0-1..c0+4 (zero off-map)
        float nbh[3][6];
        if (a.stage_tp > 0) {
#pragma unroll
            for (int dr = 0; dr < 3; ++dr) {
                const float *row = stile + (r - r0 + dr) * a.stage_tp + 4 + c0;
                const float4 m4 = *reinterpret_cast<const float4 *>(row);
                nbh[dr][0] = row[-1];
                nbh[dr][1] = m4.x; nbh[dr][2] = m4.y; nbh[dr][3] = m4.z; nbh[dr][4] = m4.w;
                nbh[dr][5] = row[4];
            }
        } else
#pragma unroll
        for (int dr = 0; dr < 3; ++dr) {
            const int rr = r + dr - 1;
            const bool rok = rr >= 0 && rr < a.H;
            const float *row = b + (long long)rr * W;
            if (vec) {
                const float4 m4 = rok ? __ldg(reinterpret_cast<const float4 *>(row + c0)) : make_float4(0.f, 0.f, 0.f, 0.f);
                nbh[dr][0] = (rok && c0 > 0) ? __ldg(row + c0 - 1) : 0.f;
                nbh[dr][1] = m4.x; nbh[dr][2] = m4.y; nbh[dr][3] = m4.z; nbh[dr][4] = m4.w;
                nbh[dr][5] = (rok && c0 + 4 < W) ? __ldg(row + c0 + 4) : 0.f;
            } else {
#pragma unroll
                for (int i = 0; i < 6; ++i) {
                    const int cc = c0 - 1 + i;
                    nbh[dr][i] = (rok && cc >= 0 && cc < W) ? __ldg(row + cc) : 0.f;
                }
            }
        }
        float bb[4];
        int sg[4];
        switch (k) {   // block-uniform: compile-time tap geometry per action
            case 0: correct_predict<0>(a, r, c0, nbh, bb, sg); break;
            case 1: correct_predict<1>(a, r, c0, nbh, bb, sg); break;
            case 2: correct_predict<2>(a, r, c0, nbh, bb, sg); break;
            case 3: correct_predict<3>(a, r, c0, nbh, bb, sg); break;
            case 4: correct_predict<4>(a, r, c0, nbh, bb, sg); break;
            case 5: correct_predict<5>(a, r, c0, nbh, bb, sg); break;
            case 6: correct_predict<6>(a, r, c0, nbh, bb, sg); break;
            case 7: correct_predict<7>(a, r, c0, nbh, bb, sg); break;
            default: correct_predict<8>(a, r, c0, nbh, bb, sg); break;
        }
        const long long x0 = (long long)r * W + c0;
        auto put = [&](int u, const float (&o)[4]) {
            float *dst = a.child + (base + u) * a.cstride + x0;
            if (a.vec_out) {
                __stcs(reinterpret_cast<float4 *>(dst), make_float4(o[0], o[1], o[2], o[3]));   // streaming
            } else {
#pragma unroll
                for (int i = 0; i < 4; ++i)
                    if (c0 + i < W) dst[i] = o[i];
            }
        };
        for (int u = 0; u < U; u += 2) {     // two children per weight load
            float o0[4], o1[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const float2 w = *reinterpret_cast<const float2 *>(&s_w[sg[i]][u]);
                o0[i] = w.x * bb[i];
                o1[i] = w.y * bb[i];
            }
            put(u, o0);
            if (u + 1 < U) put(u + 1, o1);
        }
    }
}

template <int NA>
__global__ void k_vmax(const double *__restrict__ Q, double *__restrict__ V, long long nwork, const int32_t *vmap,
                       const long long *nwork_dev = nullptr) {
    const long long w = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (w >= nwork || (nwork_dev && w >= *nwork_dev)) return;
    double best = Q[w * NA];
#pragma unroll
    for (int j = 1; j < NA; ++j) best = fmax(best, Q[w * NA + j]);
    V[vmap ? vmap[w] : w] = best + 0.0;   // +0.0 canonicalises -0 for the exact zero-padded sum
}

// one warp per parent V-node: lane j < NA backs up Q-node j over its children (ascending z, the
// oracle's order), then V = max over the lanes (exact in any order)
template <int NA>
__global__ void __launch_bounds__(256) k_backup(long long nwork, const int32_t *vmap, const double *__restrict__ R,
                                                const uint16_t *__restrict__ umask, const int32_t *__restrict__ off,
                                                const double *__restrict__ Vc, const int32_t *__restrict__ fc, int n,
                                                double gamma, double *__restrict__ Q, double *__restrict__ V,
                                                const long long *nwork_dev = nullptr) {
    const long long w = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (w >= nwork || (nwork_dev && w >= *nwork_dev)) return;
    double qv = -INFINITY;
    if (lane < NA) {
        const long long q = w * NA + lane;
        const int U = __popc((unsigned)umask[q]);
        const long long c0 = off[q];
        double acc = 0.0;
        for (int u = 0; u < U; ++u) acc += ((double)fc[c0 + u] / (double)n) * Vc[c0 + u];
        qv = R[q] + gamma * acc;                   // Alg. 6 with gamma (R13)
        Q[q] = qv;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) qv = fmax(qv, __shfl_xor_sync(0xffffffffu, qv, o));   // Alg. 7
    if (lane == 0) V[vmap ? vmap[w] : w] = qv + 0.0;
}

__global__ void k_init_roots(long long n, uint64_t *path, int32_t *root) {
    const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (i >= n) return;
    path[i] = 0;
    root[i] = (int32_t)i;
}

__global__ void k_iota_stride(int32_t *out, long long n, int r, int G) {
    const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (i < n) out[i] = (int32_t)(r + (long long)G * i);
}

// ---- host orchestration -------------------------------------------------------------------------
static inline unsigned nblk(long long n, int b) { return (unsigned)((n + b - 1) / b); }
// k_correct's shared-memory staging of the parent rows: on when the rows are 16-byte copyable and
// the CTA's rows + halo fit the default 48 KB; returns the dynamic shared memory to launch with
static size_t correct_stage(CorrectArgs &c) {
    c.vec_in = ((c.W & 3) == 0 && (c.bstride & 3) == 0 && (reinterpret_cast<uintptr_t>(c.beliefs) & 15) == 0) ? 1 : 0;
    c.vec_out = ((c.W & 3) == 0 && (c.cstride & 3) == 0 && (reinterpret_cast<uintptr_t>(c.child) & 15) == 0) ? 1 : 0;
    const bool vec = c.vec_in != 0;
    const int tp = c.W + 8;
    const size_t bytes = sizeof(float) * (size_t)(c.rows_cta + 2) * tp;
    const char *ev = std::getenv("QVTS_CORRECT_STAGE");     // read per call (tests flip it)
    const int env = ev ? std::atoi(ev) : 1;
    c.stage_tp = (env && vec && bytes <= 48 * 1024) ? tp : 0;
    return c.stage_tp ? bytes : 0;
}
// k_correct: a CTA covers ~1024 groups of 4 cells (4 passes of its 256 threads)
static inline int correct_rows_per_cta(int H, int G) {
    return std::min(H, std::max(1, 1024 / std::max(1, G)));
}

// bracket one launch with instrumentation events (no-op unless profiling is on)
#define QVTS_PROF(cat, ...)                       \
    do {                                          \
        cudaEvent_t e__;                          \
        prof_begin(m, cat, st, &e__);             \
        __VA_ARGS__;                              \
        prof_end(m, cat, st, e__);                \
    } while (0)

template <uint32_t MASK, bool LEAF>
static qvts_status launch_hist(Model &m, const BandSet &bs, const float *beliefs, long long bstride,
                               const int32_t *vmap, long long nwork, int pstride, cudaStream_t st, int *nb_eff,
                               const int32_t *skip = nullptr, const long long *nwork_dev = nullptr) {
    constexpr int NOUT = 16 * hist_cb<MASK, LEAF>() + 8;
    HistArgs a;
    a.skip = skip;
    a.nwork_dev = nwork_dev;
    a.beliefs = beliefs; a.bstride = bstride; a.vmap = vmap; a.nwork = nwork;
    a.bands = bs.bands.as<BandInfo>(); a.nb = bs.nb;
    a.entries = bs.entries.as<uint32_t>();
    a.qlist = (m.cur_leaf == QVTS_LEAF_FIB ? bs.qlist_fib : bs.qlist).as<float4>();
    a.H = m.H; a.W = m.W; a.TW = bs.tile_pitch;
    a.vec16 = ((m.W & 3) == 0 && (bstride & 3) == 0 && (reinterpret_cast<uintptr_t>(beliefs) & 15) == 0) ? 1 : 0;
    // second tile offset = 16 banks modulo 32, so the two half-warps never share a bank
    a.tstride = ((bs.tile_floats + 31) & ~31) + 16;
    a.red_off = 0;
    a.sums_off = ((2 * kRedChunk * (kHistThreads + 1)) + 3) & ~3;
    const int region = std::max(2 * a.tstride, a.sums_off + 2 * 2 * NOUT);
    a.part = m.part.as<double>(); a.pstride = pstride;
    a.skipped = m.counters.p ? m.counters.as<unsigned long long>() + 3 : nullptr;
    const size_t smem = (size_t)region * sizeof(float);
    auto kfn = nwork_dev ? k_hist<MASK, LEAF, true> : k_hist<MASK, LEAF, false>;
    QVTS_CUDA(cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    const long long nblocks = ((nwork + 1) / 2) * bs.nb;
    if (nblocks > 0x7FFFFFFFLL) { set_error("too many hist blocks"); return QVTS_ERR_INVALID_ARG; }
    QVTS_PROF(LEAF ? 0 : 1, kfn<<<(unsigned)nblocks, kPairThreads, smem, st>>>(a));
    QVTS_CUDA(cudaGetLastError());
    (LEAF ? m.pstat.leaf_cells : m.pstat.hist_cells) += nwork * m.n_free;
    *nb_eff = bs.nb;
    return QVTS_OK;
}

// leaf level on the tensor cores (leafmma.cu): one fp64 record per parent (nb = 1)
static qvts_status launch_leaf_mma_prof(Model &m, const float *beliefs, long long bstride, const int32_t *vmap,
                                        long long nwork, int pstride, cudaStream_t st, const int32_t *skip,
                                        const long long *nwork_dev) {
    QVTS_PROF(0, QVTS_TRY(launch_leaf_mma(m, beliefs, bstride, vmap, nwork, pstride, st, skip, nwork_dev)));
    m.pstat.leaf_cells += nwork * m.n_free;
    return QVTS_OK;
}

template <uint32_t MASK, bool LEAF>
static qvts_status launch_reduce(Model &m, const ReduceArgs &r, cudaStream_t st) {
    constexpr int NA = mask_count(MASK);
    const size_t smem = sizeof(double) * reduce_smem_doubles<MASK, LEAF>(r.pstride);
    auto kfn = r.xs ? k_reduce<MASK, LEAF, true> : k_reduce<MASK, LEAF, false>;
    QVTS_CUDA(cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    if (r.nwork > 0x7FFFFFFFLL) { set_error("too many parents"); return QVTS_ERR_INVALID_ARG; }
    if (r.pstride & 1) { set_error("record stride must be even (16-byte bulk copies)"); return QVTS_ERR_INVALID_ARG; }
    QVTS_PROF(LEAF ? 2 : 3, kfn<<<(unsigned)r.nwork, reduce_threads<MASK>(), smem, st>>>(r));
    QVTS_CUDA(cudaGetLastError());
    return QVTS_OK;
}

template <uint32_t MASK>
static int pstride_of(bool leaf) {
    return 16 * (leaf ? hist_cb<MASK, true>() : hist_cb<MASK, false>()) + 8;
}

template <uint32_t MASK>
static qvts_status plan_levels_t(Model &m, const RootBatch &roots, const qvts_plan_cfg &cfg, const qvts_comm *comm,
                                 cudaStream_t st, long long *nv_out) {
    constexpr int NA = mask_count(MASK);
    const int D = cfg.depth, n = cfg.n_samples;
    const bool trace = cfg.want_trace != 0;
    m.cur_leaf = cfg.leaf_bound;
    const int G = (comm && comm->nranks > 1) ? comm->nranks : 1;
    const int rank = comm ? comm->rank : 0;
    const long long shard_min = (long long)std::max(1, comm ? comm->min_nodes_per_rank : 16) * G;
    int shard_level = -1;

    VLevel &v0 = m.vl[0];
    v0.n = roots.n;
    QVTS_TRY(v0.path.ensure(sizeof(uint64_t) * roots.n));
    QVTS_TRY(v0.root.ensure(sizeof(int32_t) * roots.n));
    QVTS_TRY(v0.V.ensure(sizeof(double) * roots.n));
    QVTS_PROF(7, k_init_roots<<<nblk(roots.n, 256), 256, 0, st>>>(roots.n, v0.path.as<uint64_t>(), v0.root.as<int32_t>()));
    QVTS_CUDA(cudaGetLastError());
    QVTS_TRY(m.counters.ensure(sizeof(unsigned long long) * 4));
    QVTS_CUDA(cudaMemsetAsync(m.counters.p, 0, sizeof(unsigned long long) * 4, st));
    QVTS_TRY(m.total.ensure(sizeof(long long)));
    nv_out[0] = roots.n;

    static const char *const kLevelNames[kMaxLevels] = {"qvts level 0", "qvts level 1", "qvts level 2",
                                                         "qvts level 3", "qvts level 4", "qvts level 5",
                                                         "qvts level 6", "qvts level 7", "qvts level 8"};
    for (int d = 0; d < D; ++d) {
        NvtxRange nvtx_level(kLevelNames[d < kMaxLevels ? d : kMaxLevels - 1]);
        const bool leaf = (d == D - 1);
        VLevel &vl = m.vl[d];
        QLevel &ql = m.ql[d];
        const float *bel = d == 0 ? roots.beliefs : vl.belief.as<float>();
        const long long bstride = d == 0 ? roots.stride : m.HWp;
        // sharding: first level d >= 1 with >= shard_min V-nodes
        ql.mapped = false;
        ql.vmap_ptr = nullptr;
        long long nwork = vl.n;
        if (d == 0 && roots.active) {
            nwork = roots.n_active;
            ql.mapped = true;
            ql.vmap_ptr = roots.active;
        } else if (G > 1 && shard_level < 0 && d >= 1 && vl.n >= shard_min) {
            shard_level = d;
            nwork = vl.n > rank ? (vl.n - rank + G - 1) / G : 0;
            QVTS_TRY(ql.vmap.ensure(sizeof(int32_t) * std::max(1LL, nwork)));
            if (nwork) QVTS_PROF(7, k_iota_stride<<<nblk(nwork, 256), 256, 0, st>>>(ql.vmap.as<int32_t>(), nwork, rank, G));
            ql.mapped = true;
            ql.vmap_ptr = ql.vmap.as<int32_t>();
        }
        ql.nwork = nwork;
        const int32_t *vmap = ql.vmap_ptr;
        const long long nq = nwork * NA;
        QVTS_TRY(ql.R.ensure(sizeof(double) * std::max(1LL, nq)));
        QVTS_TRY(ql.P.ensure(sizeof(double) * 16 * std::max(1LL, nq)));
        QVTS_TRY(ql.cnt.ensure(sizeof(uint16_t) * 16 * std::max(1LL, nq)));
        QVTS_TRY(ql.umask.ensure(sizeof(uint16_t) * std::max(1LL, nq)));
        QVTS_TRY(ql.U.ensure(sizeof(int32_t) * std::max(1LL, nq)));
        QVTS_TRY(ql.off.ensure(sizeof(int32_t) * std::max(1LL, nq)));
        QVTS_TRY(ql.Q.ensure(sizeof(double) * std::max(1LL, nq)));
        if (trace) {
            QVTS_TRY(ql.zdraw.ensure((size_t)std::max(1LL, nq) * n));
            if (leaf) QVTS_TRY(ql.leafV.ensure(sizeof(double) * 16 * std::max(1LL, nq)));
        }
        if (nwork > 0) {
            // band set: a function of (level, roots) only, never of rank-local counts, so the
            // summation order -- and every value -- is identical for any number of ranks
            double expect = 1.0;    // per root: the choice must not depend on batch or wave size either
            for (int i = 0; i < d; ++i) expect *= 10.0;
            const BandSet &bs = expect < 100.0 ? m.band_small : m.band_big;
            const int pstride = pstride_of<MASK>(leaf);
            QVTS_TRY(m.part.ensure(sizeof(double) * (size_t)(nwork + 1) *
                                   std::max({bs.nb, m.leafb.nb, leaf_mma_records()}) * pstride));
            int nb_eff = bs.nb;
            ReduceArgs r;
            r.part = m.part.as<double>(); r.pstride = pstride; r.nb = bs.nb; r.nwork = nwork; r.vmap = vmap;
            r.beliefs = bel; r.bstride = bstride; r.vpath = vl.path.as<uint64_t>(); r.vroot = vl.root.as<int32_t>();
            r.root_step = roots.step_dev; r.root_ep = roots.episode_dev; r.seed = cfg.seed;
            r.level = d; r.n = n; r.O64 = m.d_O64.as<double>();
            r.ngc = m.ngc; r.gc_cell = m.d_gc_cell.as<int32_t>(); r.gc_off = m.d_gc_off.as<int32_t>();
            r.gc_val = m.d_gc_val.as<double>(); r.goal = m.goal;
            r.p_stay = m.p_stay; r.p_int = m.p_int; r.p_lat = m.p_lat; r.gamma = m.gamma;
            r.qbar = m.cur_leaf == QVTS_LEAF_FIB ? m.qbar_fib : m.qbar;
            r.R = ql.R.as<double>(); r.P = ql.P.as<double>(); r.cnt = ql.cnt.as<uint16_t>();
            r.umask = ql.umask.as<uint16_t>(); r.U = ql.U.as<int32_t>();
            r.zdraw = trace ? ql.zdraw.as<uint8_t>() : nullptr;
            r.Q = ql.Q.as<double>(); r.leafV = (trace && leaf) ? ql.leafV.as<double>() : nullptr;
            r.counters = m.counters.as<unsigned long long>();
            r.xs = nullptr; r.m8 = m.d_m8.as<uint8_t>(); r.sig = m.d_sig.as<uint8_t>(); r.W = m.W; r.acc = m.acc;
            if (cfg.sampler == QVTS_SAMPLER_ANCESTRAL) {
                // with a trace, every level keeps its state draws (qvts_trace_state_draws)
                DevBuf &xb = trace ? ql.xdraw : m.xs;
                QVTS_TRY(xb.ensure(sizeof(int32_t) * (size_t)nq * n));
                const int nch = ancestral_nch(m.HW);
                QVTS_PROF(7, k_ancestral_x<MASK><<<(unsigned)nwork, 256, sizeof(double) * (2 * nch + 1), st>>>(
                                 bel, bstride, vmap, nwork, m.HW, vl.path.as<uint64_t>(), vl.root.as<int32_t>(),
                                 roots.step_dev, roots.episode_dev, cfg.seed, d, n, xb.as<int32_t>()));
                QVTS_CUDA(cudaGetLastError());
                r.xs = xb.as<int32_t>();
            }
            if (leaf && leaf_mma_enabled(m, bstride, bel)) {
                QVTS_TRY(launch_leaf_mma_prof(m, bel, bstride, vmap, nwork, pstride, st, nullptr, nullptr));
                nb_eff = leaf_mma_records();
            } else if (leaf && leaf_kernel_supported(m)) {
                nb_eff = leaf_nsplit(m, d);
                QVTS_TRY(launch_leaf(m, bel, bstride, d == 0 ? roots.n : vl.n, vmap, nwork, nb_eff, pstride, 0, st));
            } else if (leaf) {
                QVTS_TRY((launch_hist<MASK, true>(m, bs, bel, bstride, vmap, nwork, pstride, st, &nb_eff)));
            } else {
                QVTS_TRY((launch_hist<MASK, false>(m, bs, bel, bstride, vmap, nwork, pstride, st, &nb_eff)));
            }
            r.nb = nb_eff;
            if (leaf) QVTS_TRY((launch_reduce<MASK, true>(m, r, st)));
            else QVTS_TRY((launch_reduce<MASK, false>(m, r, st)));
            QVTS_CUDA(cudaGetLastError());
        }
        if (leaf) break;
        // child offsets and count
        long long total = 0;
        if (nq > 0) {
            QVTS_PROF(4, k_scan<<<1, 1024, 0, st>>>(ql.U.as<int32_t>(), ql.off.as<int32_t>(), nq, m.total.as<long long>()));
            QVTS_CUDA(cudaGetLastError());
            QVTS_CUDA(cudaMemcpyAsync(&total, m.total.p, sizeof(long long), cudaMemcpyDeviceToHost, st));
            QVTS_CUDA(cudaStreamSynchronize(st));
        }
        VLevel &vc = m.vl[d + 1];
        vc.n = total;
        nv_out[d + 1] = total;
        const long long tn = std::max(1LL, total);
        QVTS_TRY(vc.path.ensure(sizeof(uint64_t) * tn));
        QVTS_TRY(vc.parent_q.ensure(sizeof(int32_t) * tn));
        QVTS_TRY(vc.z.ensure(sizeof(int32_t) * tn));
        QVTS_TRY(vc.f.ensure(sizeof(int32_t) * tn));
        QVTS_TRY(vc.root.ensure(sizeof(int32_t) * tn));
        QVTS_TRY(vc.V.ensure(sizeof(double) * tn));
        QVTS_TRY(vc.belief.ensure(sizeof(float) * (size_t)tn * m.HWp));
        if (nq > 0) {
            CorrectArgs c;
            c.beliefs = bel; c.bstride = bstride; c.vmap = vmap;
            c.m8 = m.d_m8.as<uint8_t>(); c.cell = m.d_cell.as<uint8_t>();
            c.O64 = m.d_O64.as<double>(); c.P = ql.P.as<double>(); c.cnt = ql.cnt.as<uint16_t>();
            c.umask = ql.umask.as<uint16_t>(); c.off = ql.off.as<int32_t>();
            c.vpath = vl.path.as<uint64_t>(); c.vroot = vl.root.as<int32_t>(); c.level = d;
            c.child = vc.belief.as<float>(); c.cstride = m.HWp;
            c.cpath = vc.path.as<uint64_t>(); c.cparent = vc.parent_q.as<int32_t>(); c.cz = vc.z.as<int32_t>();
            c.cf = vc.f.as<int32_t>(); c.croot = vc.root.as<int32_t>();
            c.H = m.H; c.W = m.W; c.G = (m.W + 3) / 4;
            c.rows_cta = correct_rows_per_cta(m.H, c.G);
            c.ntiles = (m.H + c.rows_cta - 1) / c.rows_cta;
            c.p_int = (float)m.p_int; c.p_stay = (float)m.p_stay; c.p_lat = (float)m.p_lat; c.qsel = -1;
            c.sel_q = c.sel_z = c.sel_out = nullptr;
            const long long nblocks = nq * c.ntiles;
            if (nblocks > 0x7FFFFFFFLL) { set_error("too many correct blocks"); return QVTS_ERR_INVALID_ARG; }
            const size_t csm = correct_stage(c);
            QVTS_PROF(5, k_correct<MASK><<<(unsigned)nblocks, 256, csm, st>>>(c));
            m.pstat.correct_cells_written += total * (long long)m.HW;
            QVTS_CUDA(cudaGetLastError());
        }

    }
    // S6 backup, bottom-up
    for (int d = D - 1; d >= 0; --d) {
        QLevel &ql = m.ql[d];
        VLevel &vl = m.vl[d];
        const int32_t *vmap = ql.vmap_ptr;
        if (d == shard_level) QVTS_CUDA(cudaMemsetAsync(vl.V.p, 0, sizeof(double) * std::max(1LL, vl.n), st));
        if (ql.nwork > 0) {
            if (d == D - 1) {
                QVTS_PROF(6, k_vmax<NA><<<nblk(ql.nwork, 256), 256, 0, st>>>(ql.Q.as<double>(), vl.V.as<double>(), ql.nwork, vmap));
            } else {
                VLevel &vc = m.vl[d + 1];
                QVTS_PROF(6, k_backup<NA><<<nblk(ql.nwork * 32, 256), 256, 0, st>>>(ql.nwork, vmap, ql.R.as<double>(),
                                                                  ql.umask.as<uint16_t>(), ql.off.as<int32_t>(),
                                                                  vc.V.as<double>(), vc.f.as<int32_t>(), n, m.gamma,
                                                                  ql.Q.as<double>(), vl.V.as<double>()));
            }
            QVTS_CUDA(cudaGetLastError());
        }
        if (d == shard_level) {
            // exact zero-padded sum across ranks: every rank backs up the levels above identically
            if (comm->allreduce_sum_f64(comm->ctx, vl.V.as<double>(), vl.n, (void *)st) != 0) {
                set_error("allreduce callback failed");
                return QVTS_ERR_COMM;
            }
        }
    }
    // leaf V-node count (not materialised), flagged-draw count (k_reduce) and skipped tiles
    unsigned long long cnts[4] = {0, 0, 0, 0};
    QVTS_CUDA(cudaMemcpyAsync(cnts, m.counters.p, sizeof(cnts), cudaMemcpyDeviceToHost, st));
    QVTS_CUDA(cudaStreamSynchronize(st));
    nv_out[D] = (long long)cnts[1];
    m.last_flagged = (long long)cnts[0];
    m.last_skipped = (long long)(cnts[2] + cnts[3]);
    m.last_xdraws = trace && cfg.sampler == QVTS_SAMPLER_ANCESTRAL;
    m.last_depth = D;
    m.last_shard_level = shard_level;
    m.last_n = n;
    m.last_trace = trace;
    return QVTS_OK;
}

// ---- graph-captured plan step (small trees) ------------------------------------------------------
// The same kernels as plan_levels_t, with every level's V-node count kept on the device
// (m.lvl_cnt[d], written by k_scan) and grids sized for the worst case Vmax[d] (children per
// Q-node <= min(n, 16)), so one plan step is a fixed launch sequence that a CUDA graph replays
// with no host synchronisation between levels.  Used for single-root plan steps whose worst-case
// tree fits kGraphBudget; results are bit-identical to plan_levels_t (same kernels, same order).
constexpr double kGraphBudget = 2.0e9;    // bytes of worst-case materialised beliefs

__global__ void k_set_count(long long *cnt, long long v) { cnt[0] = v; }

static bool graph_eligible(const Model &m, const qvts_plan_cfg &cfg, long long *vmax) {
    vmax[0] = 1;
    double bytes = 0.0;
    for (int d = 0; d < cfg.depth; ++d) {
        vmax[d + 1] = vmax[d] * m.NA * std::min(cfg.n_samples, 16);
        if (d + 1 < cfg.depth) bytes += (double)vmax[d + 1] * m.HWp * 4.0;
        if (vmax[d + 1] > (1LL << 26)) return false;
    }
    return bytes <= kGraphBudget;
}

template <uint32_t MASK>
static qvts_status plan_levels_dev_t(Model &m, const float *root, const qvts_plan_cfg &cfg, const long long *vmax,
                                     cudaStream_t st) {
    constexpr int NA = mask_count(MASK);
    const int D = cfg.depth, n = cfg.n_samples;
    long long *cnt = m.lvl_cnt.as<long long>();           // [D+1] V-node counts per level
    VLevel &v0 = m.vl[0];
    QVTS_PROF(7, k_init_roots<<<1, 256, 0, st>>>(1, v0.path.as<uint64_t>(), v0.root.as<int32_t>()));
    QVTS_PROF(7, k_set_count<<<1, 1, 0, st>>>(cnt, 1));
    QVTS_CUDA(cudaMemsetAsync(m.counters.p, 0, sizeof(unsigned long long) * 4, st));
    for (int d = 0; d < D; ++d) {
        const bool leaf = (d == D - 1);
        VLevel &vl = m.vl[d];
        QLevel &ql = m.ql[d];
        ql.nwork = vmax[d];
        ql.mapped = false;
        ql.vmap_ptr = nullptr;
        const float *bel = d == 0 ? root : vl.belief.as<float>();
        const long long bstride = d == 0 ? m.HW : m.HWp;
        const long long nwork = vmax[d], nq = nwork * NA;
        double expect = 1.0;
        for (int i = 0; i < d; ++i) expect *= 10.0;
        const BandSet &bs = expect < 100.0 ? m.band_small : m.band_big;
        const int pstride = pstride_of<MASK>(leaf);
        ReduceArgs r;
        r.part = m.part.as<double>(); r.pstride = pstride; r.nb = bs.nb; r.nwork = nwork; r.vmap = nullptr;
        r.beliefs = bel; r.bstride = bstride; r.vpath = vl.path.as<uint64_t>(); r.vroot = vl.root.as<int32_t>();
        r.root_step = m.ep_root_step.as<uint32_t>(); r.root_ep = m.ep_root_ep.as<uint32_t>(); r.seed = cfg.seed;
        r.level = d; r.n = n; r.O64 = m.d_O64.as<double>();
        r.ngc = m.ngc; r.gc_cell = m.d_gc_cell.as<int32_t>(); r.gc_off = m.d_gc_off.as<int32_t>();
        r.gc_val = m.d_gc_val.as<double>(); r.goal = m.goal;
        r.p_stay = m.p_stay; r.p_int = m.p_int; r.p_lat = m.p_lat; r.gamma = m.gamma;
        r.qbar = m.cur_leaf == QVTS_LEAF_FIB ? m.qbar_fib : m.qbar;
        r.R = ql.R.as<double>(); r.P = ql.P.as<double>(); r.cnt = ql.cnt.as<uint16_t>();
        r.umask = ql.umask.as<uint16_t>(); r.U = ql.U.as<int32_t>(); r.zdraw = nullptr;
        r.Q = ql.Q.as<double>(); r.leafV = nullptr;
        r.counters = m.counters.as<unsigned long long>();
        r.xs = nullptr; r.m8 = m.d_m8.as<uint8_t>(); r.sig = m.d_sig.as<uint8_t>(); r.W = m.W; r.acc = m.acc;
        r.nwork_dev = cnt + d;
        if (cfg.sampler == QVTS_SAMPLER_ANCESTRAL) {
            const int nch = ancestral_nch(m.HW);
            QVTS_PROF(7, k_ancestral_x<MASK><<<(unsigned)nwork, 256, sizeof(double) * (2 * nch + 1), st>>>(
                             bel, bstride, nullptr, nwork, m.HW, vl.path.as<uint64_t>(), vl.root.as<int32_t>(),
                             r.root_step, r.root_ep, cfg.seed, d, n, m.xs.as<int32_t>(), nullptr, cnt + d));
            r.xs = m.xs.as<int32_t>();
        }
        int nb_eff = bs.nb;
        if (leaf && leaf_mma_enabled(m, bstride, bel)) {
            QVTS_TRY(launch_leaf_mma_prof(m, bel, bstride, nullptr, nwork, pstride, st, nullptr, cnt + d));
            nb_eff = leaf_mma_records();
        } else if (leaf && leaf_kernel_supported(m)) {
            nb_eff = leaf_nsplit(m, d);
            QVTS_TRY(launch_leaf(m, bel, bstride, std::max(1LL, vmax[d]), nullptr, nwork, nb_eff, pstride, 0, st, cnt + d));
        } else if (leaf) {
            QVTS_TRY((launch_hist<MASK, true>(m, bs, bel, bstride, nullptr, nwork, pstride, st, &nb_eff, nullptr, cnt + d)));
        } else {
            QVTS_TRY((launch_hist<MASK, false>(m, bs, bel, bstride, nullptr, nwork, pstride, st, &nb_eff, nullptr, cnt + d)));
        }
        r.nb = nb_eff;
        if (leaf) QVTS_TRY((launch_reduce<MASK, true>(m, r, st)));
        else QVTS_TRY((launch_reduce<MASK, false>(m, r, st)));
        if (leaf) break;
        QVTS_PROF(4, k_scan<<<1, 1024, 0, st>>>(ql.U.as<int32_t>(), ql.off.as<int32_t>(), nq, cnt + d + 1, nullptr,
                                               cnt + d, NA));
        VLevel &vc = m.vl[d + 1];
        CorrectArgs c;
        c.beliefs = bel; c.bstride = bstride; c.vmap = nullptr;
        c.m8 = m.d_m8.as<uint8_t>(); c.cell = m.d_cell.as<uint8_t>();
        c.O64 = m.d_O64.as<double>(); c.P = ql.P.as<double>(); c.cnt = ql.cnt.as<uint16_t>();
        c.umask = ql.umask.as<uint16_t>(); c.off = ql.off.as<int32_t>();
        c.vpath = vl.path.as<uint64_t>(); c.vroot = vl.root.as<int32_t>(); c.level = d;
        c.child = vc.belief.as<float>(); c.cstride = m.HWp;
        c.cpath = vc.path.as<uint64_t>(); c.cparent = vc.parent_q.as<int32_t>(); c.cz = vc.z.as<int32_t>();
        c.cf = vc.f.as<int32_t>(); c.croot = vc.root.as<int32_t>();
        c.H = m.H; c.W = m.W; c.G = (m.W + 3) / 4;
        c.rows_cta = correct_rows_per_cta(m.H, c.G);
        c.ntiles = (m.H + c.rows_cta - 1) / c.rows_cta;
        c.p_int = (float)m.p_int; c.p_stay = (float)m.p_stay; c.p_lat = (float)m.p_lat; c.qsel = -1;
        c.sel_q = c.sel_z = c.sel_out = nullptr;
        c.nwork_dev = cnt + d;
        { const size_t csm_ = correct_stage(c);
        QVTS_PROF(5, k_correct<MASK><<<(unsigned)(nq * c.ntiles), 256, csm_, st>>>(c)); }
    }
    for (int d = D - 1; d >= 0; --d) {
        QLevel &ql = m.ql[d];
        VLevel &vl = m.vl[d];
        if (d == D - 1) {
            QVTS_PROF(6, k_vmax<NA><<<nblk(vmax[d], 256), 256, 0, st>>>(ql.Q.as<double>(), vl.V.as<double>(), vmax[d],
                                                                        nullptr, cnt + d));
        } else {
            VLevel &vc = m.vl[d + 1];
            QVTS_PROF(6, k_backup<NA><<<nblk(vmax[d] * 32, 256), 256, 0, st>>>(
                             vmax[d], nullptr, ql.R.as<double>(), ql.umask.as<uint16_t>(), ql.off.as<int32_t>(),
                             vc.V.as<double>(), vc.f.as<int32_t>(), n, m.gamma, ql.Q.as<double>(), vl.V.as<double>(),
                             cnt + d));
        }
    }
    QVTS_CUDA(cudaGetLastError());
    return QVTS_OK;
}

// workspace for the worst-case tree (outside any capture: ensure() may allocate)
template <uint32_t MASK>
static qvts_status plan_dev_prepare_t(Model &m, const qvts_plan_cfg &cfg, const long long *vmax) {
    constexpr int NA = mask_count(MASK);
    const int D = cfg.depth;
    QVTS_TRY(m.lvl_cnt.ensure(sizeof(long long) * (kMaxLevels + 1)));
    QVTS_TRY(m.counters.ensure(sizeof(unsigned long long) * 4));
    QVTS_TRY(m.total.ensure(sizeof(long long)));
    size_t part = 0;
    for (int d = 0; d <= D; ++d) {
        VLevel &vl = m.vl[d];
        const long long tn = std::max(1LL, vmax[d]);
        QVTS_TRY(vl.path.ensure(sizeof(uint64_t) * tn));
        QVTS_TRY(vl.root.ensure(sizeof(int32_t) * tn));
        QVTS_TRY(vl.V.ensure(sizeof(double) * tn));
        if (d >= 1) {
            QVTS_TRY(vl.parent_q.ensure(sizeof(int32_t) * tn));
            QVTS_TRY(vl.z.ensure(sizeof(int32_t) * tn));
            QVTS_TRY(vl.f.ensure(sizeof(int32_t) * tn));
            if (d < D) QVTS_TRY(vl.belief.ensure(sizeof(float) * (size_t)tn * m.HWp));
        }
        if (d < D) {
            QLevel &ql = m.ql[d];
            const long long nq = tn * NA;
            QVTS_TRY(ql.R.ensure(sizeof(double) * nq));
            QVTS_TRY(ql.P.ensure(sizeof(double) * 16 * nq));
            QVTS_TRY(ql.cnt.ensure(sizeof(uint16_t) * 16 * nq));
            QVTS_TRY(ql.umask.ensure(sizeof(uint16_t) * nq));
            QVTS_TRY(ql.U.ensure(sizeof(int32_t) * nq));
            QVTS_TRY(ql.off.ensure(sizeof(int32_t) * nq));
            QVTS_TRY(ql.Q.ensure(sizeof(double) * nq));
            double expect = 1.0;
            for (int i = 0; i < d; ++i) expect *= 10.0;
            const BandSet &bs = expect < 100.0 ? m.band_small : m.band_big;
            part = std::max(part, sizeof(double) * (size_t)(tn + 1) *
                                      std::max({bs.nb, m.leafb.nb, leaf_mma_records()}) * pstride_of<MASK>(d == D - 1));
            if (cfg.sampler == QVTS_SAMPLER_ANCESTRAL)
                QVTS_TRY(m.xs.ensure(sizeof(int32_t) * (size_t)nq * cfg.n_samples));
        }
    }
    QVTS_TRY(m.part.ensure(part));
    return QVTS_OK;
}

template <uint32_t MASK>
static qvts_status root_marginals_t(Model &m, const RootBatch &roots, cudaStream_t st) {
    constexpr int NA = mask_count(MASK);
    VLevel &v0 = m.vl[0];
    QLevel &ql = m.ql[0];
    v0.n = roots.n;
    QVTS_TRY(v0.path.ensure(sizeof(uint64_t) * roots.n));
    QVTS_TRY(v0.root.ensure(sizeof(int32_t) * roots.n));
    QVTS_PROF(7, k_init_roots<<<nblk(roots.n, 256), 256, 0, st>>>(roots.n, v0.path.as<uint64_t>(), v0.root.as<int32_t>()));
    const long long nwork = roots.active ? roots.n_active : roots.n;
    ql.nwork = nwork;
    ql.mapped = roots.active != nullptr;
    ql.vmap_ptr = roots.active;
    if (nwork == 0) return QVTS_OK;
    const long long nq = nwork * NA;
    QVTS_TRY(ql.R.ensure(sizeof(double) * nq));
    QVTS_TRY(ql.P.ensure(sizeof(double) * 16 * nq));
    QVTS_TRY(ql.cnt.ensure(sizeof(uint16_t) * 16 * nq));
    QVTS_TRY(ql.umask.ensure(sizeof(uint16_t) * nq));
    QVTS_TRY(ql.U.ensure(sizeof(int32_t) * nq));
    const BandSet &bs = m.band_small;     // the level-0 band set of plan_levels (same sums)
    const int pstride = pstride_of<MASK>(false);
    QVTS_TRY(m.part.ensure(sizeof(double) * (size_t)(nwork + 1) * bs.nb * pstride));
    int nb_eff = bs.nb;
    QVTS_TRY((launch_hist<MASK, false>(m, bs, roots.beliefs, roots.stride, roots.active, nwork, pstride, st, &nb_eff)));
    ReduceArgs r;
    std::memset(&r, 0, sizeof(r));
    r.part = m.part.as<double>(); r.pstride = pstride; r.nb = nb_eff; r.nwork = nwork; r.vmap = roots.active;
    r.beliefs = roots.beliefs; r.bstride = roots.stride; r.vpath = v0.path.as<uint64_t>(); r.vroot = v0.root.as<int32_t>();
    r.root_step = roots.step_dev; r.root_ep = roots.episode_dev; r.n = 1; r.O64 = m.d_O64.as<double>();
    r.ngc = m.ngc; r.gc_cell = m.d_gc_cell.as<int32_t>(); r.gc_off = m.d_gc_off.as<int32_t>();
    r.gc_val = m.d_gc_val.as<double>(); r.goal = m.goal; r.p_stay = m.p_stay; r.p_int = m.p_int; r.p_lat = m.p_lat;
    r.gamma = m.gamma; r.acc = m.acc; r.R = ql.R.as<double>(); r.P = ql.P.as<double>(); r.cnt = ql.cnt.as<uint16_t>();
    r.umask = ql.umask.as<uint16_t>(); r.U = ql.U.as<int32_t>();
    return launch_reduce<MASK, false>(m, r, st);
}

template <uint32_t MASK>
static qvts_status correct_selected_t(Model &m, const RootBatch &roots, const int32_t *sel_q, const int32_t *sel_z,
                                      const int32_t *sel_out, long long n, float *out, long long ostride,
                                      cudaStream_t st) {
    if (n == 0) return QVTS_OK;
    CorrectArgs c;
    std::memset(&c, 0, sizeof(c));
    c.beliefs = roots.beliefs; c.bstride = roots.stride; c.vmap = m.ql[0].vmap_ptr;
    c.m8 = m.d_m8.as<uint8_t>(); c.cell = m.d_cell.as<uint8_t>(); c.O64 = m.d_O64.as<double>();
    c.P = m.ql[0].P.as<double>(); c.cnt = m.ql[0].cnt.as<uint16_t>();
    c.child = out; c.cstride = ostride; c.H = m.H; c.W = m.W; c.G = (m.W + 3) / 4;
    c.rows_cta = correct_rows_per_cta(m.H, c.G);
    c.ntiles = (m.H + c.rows_cta - 1) / c.rows_cta;
    c.p_int = (float)m.p_int; c.p_stay = (float)m.p_stay; c.p_lat = (float)m.p_lat; c.qsel = -1;
    c.sel_q = sel_q; c.sel_z = sel_z; c.sel_out = sel_out;
    { const size_t csm_ = correct_stage(c);
    QVTS_PROF(5, k_correct<MASK><<<(unsigned)(n * c.ntiles), 256, csm_, st>>>(c)); }
    QVTS_CUDA(cudaGetLastError());
    return QVTS_OK;
}

// ---- explicit V-node batches (best-first QVTS, bestfirst.cu) --------------------------------------
// S1-S3 of `nwork` V-nodes of one level (the same kernels and Philox keys as plan_levels), then the
// exclusive child offsets; *total = number of children (synchronises `st`).
template <uint32_t MASK>
static qvts_status expand_marginals_t(Model &m, const ExpandSpec &e, QLevel &ql, cudaStream_t st, long long *total) {
    constexpr int NA = mask_count(MASK);
    const long long nwork = e.nwork, nq = nwork * NA;
    ql.nwork = nwork;
    ql.mapped = false;
    ql.vmap_ptr = nullptr;
    QVTS_TRY(ql.R.ensure(sizeof(double) * nq));
    QVTS_TRY(ql.P.ensure(sizeof(double) * 16 * nq));
    QVTS_TRY(ql.cnt.ensure(sizeof(uint16_t) * 16 * nq));
    QVTS_TRY(ql.umask.ensure(sizeof(uint16_t) * nq));
    QVTS_TRY(ql.U.ensure(sizeof(int32_t) * nq));
    QVTS_TRY(ql.off.ensure(sizeof(int32_t) * nq));
    QVTS_TRY(ql.Q.ensure(sizeof(double) * nq));
    QVTS_TRY(m.counters.ensure(sizeof(unsigned long long) * 4));
    QVTS_TRY(m.total.ensure(sizeof(long long)));
    const BandSet &bs = m.band_small;
    const int pstride = pstride_of<MASK>(false);
    QVTS_TRY(m.part.ensure(sizeof(double) * (size_t)(nwork + 1) * bs.nb * pstride));
    ReduceArgs r;
    std::memset(&r, 0, sizeof(r));
    r.part = m.part.as<double>(); r.pstride = pstride; r.nb = bs.nb; r.nwork = nwork; r.vmap = nullptr;
    r.beliefs = e.beliefs; r.bstride = e.bstride; r.vpath = e.vpath; r.vroot = e.vroot;
    r.root_step = e.root_step; r.root_ep = e.root_ep; r.seed = e.seed; r.level = e.level; r.n = e.n;
    r.O64 = m.d_O64.as<double>(); r.ngc = m.ngc; r.gc_cell = m.d_gc_cell.as<int32_t>();
    r.gc_off = m.d_gc_off.as<int32_t>(); r.gc_val = m.d_gc_val.as<double>(); r.goal = m.goal;
    r.p_stay = m.p_stay; r.p_int = m.p_int; r.p_lat = m.p_lat; r.gamma = m.gamma;
    r.R = ql.R.as<double>(); r.P = ql.P.as<double>(); r.cnt = ql.cnt.as<uint16_t>();
    r.umask = ql.umask.as<uint16_t>(); r.U = ql.U.as<int32_t>(); r.Q = ql.Q.as<double>();
    r.counters = m.counters.as<unsigned long long>();
    r.m8 = m.d_m8.as<uint8_t>(); r.sig = m.d_sig.as<uint8_t>(); r.W = m.W; r.acc = m.acc;
    if (e.sampler == QVTS_SAMPLER_ANCESTRAL) {
        QVTS_TRY(m.xs.ensure(sizeof(int32_t) * (size_t)nq * e.n));
        const int nch = ancestral_nch(m.HW);
        QVTS_PROF(7, k_ancestral_x<MASK><<<(unsigned)nwork, 256, sizeof(double) * (2 * nch + 1), st>>>(
                         e.beliefs, e.bstride, nullptr, nwork, m.HW, e.vpath, e.vroot, e.root_step, e.root_ep,
                         e.seed, e.level, e.n, m.xs.as<int32_t>()));
        QVTS_CUDA(cudaGetLastError());
        r.xs = m.xs.as<int32_t>();
    }
    int nb_eff = bs.nb;
    QVTS_TRY((launch_hist<MASK, false>(m, bs, e.beliefs, e.bstride, nullptr, nwork, pstride, st, &nb_eff)));
    r.nb = nb_eff;
    QVTS_TRY((launch_reduce<MASK, false>(m, r, st)));
    QVTS_PROF(4, k_scan<<<1, 1024, 0, st>>>(ql.U.as<int32_t>(), ql.off.as<int32_t>(), nq, m.total.as<long long>()));
    QVTS_CUDA(cudaGetLastError());
    QVTS_CUDA(cudaMemcpyAsync(total, m.total.p, sizeof(long long), cudaMemcpyDeviceToHost, st));
    QVTS_CUDA(cudaStreamSynchronize(st));
    return QVTS_OK;
}

// S4 of the batch prepared by expand_marginals: child j of Q-node q lands at off[q] + j.
template <uint32_t MASK>
static qvts_status expand_children_t(Model &m, const ExpandSpec &e, const QLevel &ql, const ChildOut &o,
                                     cudaStream_t st) {
    constexpr int NA = mask_count(MASK);
    CorrectArgs c;
    std::memset(&c, 0, sizeof(c));
    c.beliefs = e.beliefs; c.bstride = e.bstride; c.vmap = nullptr;
    c.m8 = m.d_m8.as<uint8_t>(); c.cell = m.d_cell.as<uint8_t>();
    c.O64 = m.d_O64.as<double>(); c.P = ql.P.as<double>(); c.cnt = ql.cnt.as<uint16_t>();
    c.umask = ql.umask.as<uint16_t>(); c.off = ql.off.as<int32_t>();
    c.vpath = e.vpath; c.vroot = e.vroot; c.level = e.level;
    c.child = o.belief; c.cstride = o.stride;
    c.cpath = o.path; c.cparent = o.parent_q; c.cz = o.z; c.cf = o.f; c.croot = o.root;
    c.H = m.H; c.W = m.W; c.G = (m.W + 3) / 4;
    c.rows_cta = correct_rows_per_cta(m.H, c.G);
    c.ntiles = (m.H + c.rows_cta - 1) / c.rows_cta;
    c.p_int = (float)m.p_int; c.p_stay = (float)m.p_stay; c.p_lat = (float)m.p_lat; c.qsel = -1;
    const long long nblocks = e.nwork * NA * c.ntiles;
    if (nblocks > 0x7FFFFFFFLL) { set_error("too many correct blocks"); return QVTS_ERR_INVALID_ARG; }
    { const size_t csm_ = correct_stage(c);
    QVTS_PROF(5, k_correct<MASK><<<(unsigned)nblocks, 256, csm_, st>>>(c)); }
    QVTS_CUDA(cudaGetLastError());
    return QVTS_OK;
}

// One best-first expansion with every index on the device, so the launches can be captured in a
// CUDA graph: the V-node *L.sel of the pool (its level read from its path) gets S1-S3, the child
// offsets (*L.total = child count) and S4 into the pool at *L.cbase + off; while *L.skip is set
// every launch returns at once.
template <uint32_t MASK>
static qvts_status bf_expand_launch_t(Model &m, const BfLaunch &L, QLevel &ql, cudaStream_t st) {
    constexpr int NA = mask_count(MASK);
    const BandSet &bs = m.band_small;
    const int pstride = pstride_of<MASK>(false);
    ReduceArgs r;
    std::memset(&r, 0, sizeof(r));
    r.part = m.part.as<double>(); r.pstride = pstride; r.nb = bs.nb; r.nwork = 1; r.vmap = L.sel;
    r.beliefs = L.bel; r.bstride = L.stride; r.vpath = L.path; r.vroot = L.root;
    r.root_step = L.root_step; r.root_ep = L.root_ep; r.seed = L.seed; r.level = -1; r.n = L.n;
    r.O64 = m.d_O64.as<double>(); r.ngc = m.ngc; r.gc_cell = m.d_gc_cell.as<int32_t>();
    r.gc_off = m.d_gc_off.as<int32_t>(); r.gc_val = m.d_gc_val.as<double>(); r.goal = m.goal;
    r.p_stay = m.p_stay; r.p_int = m.p_int; r.p_lat = m.p_lat; r.gamma = m.gamma;
    r.R = ql.R.as<double>(); r.P = ql.P.as<double>(); r.cnt = ql.cnt.as<uint16_t>();
    r.umask = ql.umask.as<uint16_t>(); r.U = ql.U.as<int32_t>(); r.Q = ql.Q.as<double>();
    r.counters = m.counters.as<unsigned long long>();
    r.m8 = m.d_m8.as<uint8_t>(); r.sig = m.d_sig.as<uint8_t>(); r.W = m.W; r.acc = m.acc;
    r.skip = L.skip;
    if (L.sampler == QVTS_SAMPLER_ANCESTRAL) {
        const int nch = ancestral_nch(m.HW);
        QVTS_PROF(7, k_ancestral_x<MASK><<<1, 256, sizeof(double) * (2 * nch + 1), st>>>(
                         L.bel, L.stride, L.sel, 1, m.HW, L.path, L.root, L.root_step, L.root_ep, L.seed, -1, L.n,
                         m.xs.as<int32_t>(), L.skip));
        QVTS_CUDA(cudaGetLastError());
        r.xs = m.xs.as<int32_t>();
    }
    int nb_eff = bs.nb;
    QVTS_TRY((launch_hist<MASK, false>(m, bs, L.bel, L.stride, L.sel, 1, pstride, st, &nb_eff, L.skip)));
    r.nb = nb_eff;
    QVTS_TRY((launch_reduce<MASK, false>(m, r, st)));
    QVTS_PROF(4, k_scan<<<1, 1024, 0, st>>>(ql.U.as<int32_t>(), ql.off.as<int32_t>(), NA, L.total, L.skip));
    QVTS_CUDA(cudaGetLastError());
    CorrectArgs c;
    std::memset(&c, 0, sizeof(c));
    c.beliefs = L.bel; c.bstride = L.stride; c.vmap = L.sel;
    c.m8 = m.d_m8.as<uint8_t>(); c.cell = m.d_cell.as<uint8_t>();
    c.O64 = m.d_O64.as<double>(); c.P = ql.P.as<double>(); c.cnt = ql.cnt.as<uint16_t>();
    c.umask = ql.umask.as<uint16_t>(); c.off = ql.off.as<int32_t>();
    c.vpath = L.path; c.vroot = L.root; c.level = -1;
    c.child = L.bel; c.cstride = L.stride;
    c.cpath = L.path; c.cparent = L.pq; c.cz = L.z; c.cf = L.f; c.croot = L.root;
    c.H = m.H; c.W = m.W; c.G = (m.W + 3) / 4;
    c.rows_cta = correct_rows_per_cta(m.H, c.G);
    c.ntiles = (m.H + c.rows_cta - 1) / c.rows_cta;
    c.p_int = (float)m.p_int; c.p_stay = (float)m.p_stay; c.p_lat = (float)m.p_lat; c.qsel = -1;
    c.skip = L.skip; c.cbase_dev = L.cbase;
    { const size_t csm_ = correct_stage(c);
    QVTS_PROF(5, k_correct<MASK><<<(unsigned)(NA * c.ntiles), 256, csm_, st>>>(c)); }
    QVTS_CUDA(cudaGetLastError());
    return QVTS_OK;
}

qvts_status bf_expand_prepare(Model &m, QLevel &ql, int n, int sampler) {
    const long long nq = m.NA;
    QVTS_TRY(ql.R.ensure(sizeof(double) * nq));
    QVTS_TRY(ql.P.ensure(sizeof(double) * 16 * nq));
    QVTS_TRY(ql.cnt.ensure(sizeof(uint16_t) * 16 * nq));
    QVTS_TRY(ql.umask.ensure(sizeof(uint16_t) * nq));
    QVTS_TRY(ql.U.ensure(sizeof(int32_t) * nq));
    QVTS_TRY(ql.off.ensure(sizeof(int32_t) * nq));
    QVTS_TRY(ql.Q.ensure(sizeof(double) * nq));
    QVTS_TRY(m.counters.ensure(sizeof(unsigned long long) * 4));
    int pstride = 0;
#define QVTS_PS(MASK) pstride = pstride_of<MASK>(false)
    QVTS_DISPATCH_MASK(m.mask, QVTS_PS);
#undef QVTS_PS
    QVTS_TRY(m.part.ensure(sizeof(double) * 2 * m.band_small.nb * pstride));
    if (sampler == QVTS_SAMPLER_ANCESTRAL) QVTS_TRY(m.xs.ensure(sizeof(int32_t) * (size_t)nq * n));
    return QVTS_OK;
}

qvts_status bf_expand_launch(Model &m, const BfLaunch &L, QLevel &ql, cudaStream_t st) {
    qvts_status s = QVTS_ERR_INVALID_ARG;
#define QVTS_BL(MASK) s = bf_expand_launch_t<MASK>(m, L, ql, st)
    QVTS_DISPATCH_MASK(m.mask, QVTS_BL);
#undef QVTS_BL
    return s;
}

qvts_status expand_marginals(Model &m, const ExpandSpec &e, QLevel &ql, cudaStream_t st, long long *total) {
    qvts_status s = QVTS_ERR_INVALID_ARG;
#define QVTS_EM(MASK) s = expand_marginals_t<MASK>(m, e, ql, st, total)
    QVTS_DISPATCH_MASK(m.mask, QVTS_EM);
#undef QVTS_EM
    return s;
}

qvts_status expand_children(Model &m, const ExpandSpec &e, const QLevel &ql, const ChildOut &o, cudaStream_t st) {
    qvts_status s = QVTS_ERR_INVALID_ARG;
#define QVTS_EC(MASK) s = expand_children_t<MASK>(m, e, ql, o, st)
    QVTS_DISPATCH_MASK(m.mask, QVTS_EC);
#undef QVTS_EC
    return s;
}

qvts_status root_marginals(Model &m, const RootBatch &roots, cudaStream_t st) {
    qvts_status s = QVTS_ERR_INVALID_ARG;
#define QVTS_RM(MASK) s = root_marginals_t<MASK>(m, roots, st)
    QVTS_DISPATCH_MASK(m.mask, QVTS_RM);
#undef QVTS_RM
    return s;
}

qvts_status correct_selected(Model &m, const RootBatch &roots, const int32_t *sel_q, const int32_t *sel_z,
                             const int32_t *sel_out, long long n, float *out, long long ostride, cudaStream_t st) {
    qvts_status s = QVTS_ERR_INVALID_ARG;
#define QVTS_CS(MASK) s = correct_selected_t<MASK>(m, roots, sel_q, sel_z, sel_out, n, out, ostride, st)
    QVTS_DISPATCH_MASK(m.mask, QVTS_CS);
#undef QVTS_CS
    return s;
}

static qvts_status plan_dev_prepare(Model &m, const qvts_plan_cfg &cfg, const long long *vmax) {
    qvts_status s = QVTS_ERR_INVALID_ARG;
#define QVTS_PDP(MASK) s = plan_dev_prepare_t<MASK>(m, cfg, vmax)
    QVTS_DISPATCH_MASK(m.mask, QVTS_PDP);
#undef QVTS_PDP
    return s;
}

static qvts_status plan_levels_dev(Model &m, const float *root, const qvts_plan_cfg &cfg, const long long *vmax,
                                   cudaStream_t st) {
    qvts_status s = QVTS_ERR_INVALID_ARG;
#define QVTS_PLD(MASK) s = plan_levels_dev_t<MASK>(m, root, cfg, vmax, st)
    QVTS_DISPATCH_MASK(m.mask, QVTS_PLD);
#undef QVTS_PLD
    return s;
}

// One graph-captured plan step (see plan_levels_dev_t): root copied into a private buffer, keys
// uploaded, the cached graph replayed (re-captured when the configuration or a buffer changed), then
// Q(root, .), the level counts and the counters read back with one synchronisation.
static qvts_status plan_step_graph(Model &m, const float *root_dev, const qvts_plan_cfg &cfg, const long long *vmax,
                                   cudaStream_t cst, double *q, long long *nv) {
    if (!m.pg_stream) QVTS_CUDA(cudaStreamCreateWithFlags(&m.pg_stream, cudaStreamNonBlocking));
    if (!m.pg_join) QVTS_CUDA(cudaEventCreateWithFlags(&m.pg_join, cudaEventDisableTiming));
    cudaStream_t st = m.pg_stream;
    QVTS_CUDA(cudaEventRecord(m.pg_join, cst));
    QVTS_CUDA(cudaStreamWaitEvent(st, m.pg_join, 0));
    m.cur_leaf = cfg.leaf_bound;
    QVTS_TRY(plan_dev_prepare(m, cfg, vmax));
    QVTS_TRY(m.root_buf.ensure(sizeof(float) * (size_t)m.HWp));
    QVTS_CUDA(cudaMemcpyAsync(m.root_buf.p, root_dev, sizeof(float) * m.HW, cudaMemcpyDeviceToDevice, st));
    uint32_t keys[2] = {cfg.step, cfg.episode};
    QVTS_CUDA(cudaMemcpyAsync(m.ep_root_step.p, &keys[0], sizeof(uint32_t), cudaMemcpyHostToDevice, st));
    QVTS_CUDA(cudaMemcpyAsync(m.ep_root_ep.p, &keys[1], sizeof(uint32_t), cudaMemcpyHostToDevice, st));
    std::vector<uintptr_t> key = {(uintptr_t)cfg.depth, (uintptr_t)cfg.n_samples, (uintptr_t)cfg.seed,
                                  (uintptr_t)cfg.sampler, (uintptr_t)cfg.leaf_bound, (uintptr_t)m.part.p,
                                  (uintptr_t)m.lvl_cnt.p, (uintptr_t)m.counters.p, (uintptr_t)m.root_buf.p,
                                  (uintptr_t)m.xs.p, (uintptr_t)m.ep_root_step.p, (uintptr_t)m.ep_root_ep.p};
    // the leaf offset qbar is a kernel argument captured by value: a later value / FIB iteration
    // with another qbar (or rebuilt Q' lists) must re-capture
    uint64_t qb_bits[2];
    std::memcpy(&qb_bits[0], &m.qbar, sizeof(double));
    std::memcpy(&qb_bits[1], &m.qbar_fib, sizeof(double));
    key.push_back((uintptr_t)qb_bits[0]);
    key.push_back((uintptr_t)qb_bits[1]);
    for (const DevBuf *b : {&m.band_big.qlist, &m.band_big.qlist_fib, &m.band_small.qlist, &m.band_small.qlist_fib,
                            &m.leafb.qlist, &m.leafb.qlist_fib})
        key.push_back((uintptr_t)b->p);
    for (int d = 0; d <= cfg.depth; ++d) {
        const VLevel &vl = m.vl[d];
        for (const DevBuf *b : {&vl.path, &vl.parent_q, &vl.z, &vl.f, &vl.root, &vl.V, &vl.belief}) key.push_back((uintptr_t)b->p);
        if (d < cfg.depth) {
            const QLevel &ql = m.ql[d];
            for (const DevBuf *b : {&ql.R, &ql.P, &ql.cnt, &ql.umask, &ql.U, &ql.off, &ql.Q}) key.push_back((uintptr_t)b->p);
        }
    }
    if (!m.pg_exec || key != m.pg_key) {
        if (m.pg_exec) { cudaGraphExecDestroy(m.pg_exec); m.pg_exec = nullptr; }
        cudaGraph_t graph;
        QVTS_CUDA(cudaStreamBeginCapture(st, cudaStreamCaptureModeRelaxed));
        const qvts_status s2 = plan_levels_dev(m, m.root_buf.as<float>(), cfg, vmax, st);
        const cudaError_t e = cudaStreamEndCapture(st, &graph);
        QVTS_TRY(s2);
        QVTS_CUDA(e);
        const cudaError_t e2 = cudaGraphInstantiate(&m.pg_exec, graph, 0);
        cudaGraphDestroy(graph);
        QVTS_CUDA(e2);
        m.pg_key = key;
    }
    QVTS_CUDA(cudaEventRecord(m.ev0, st));
    QVTS_CUDA(cudaGraphLaunch(m.pg_exec, st));
    QVTS_CUDA(cudaEventRecord(m.ev1, st));
    long long cnt[kMaxLevels + 1];
    unsigned long long ctr[4];
    QVTS_CUDA(cudaMemcpyAsync(q, m.ql[0].Q.p, sizeof(double) * m.NA, cudaMemcpyDeviceToHost, st));
    QVTS_CUDA(cudaMemcpyAsync(cnt, m.lvl_cnt.p, sizeof(long long) * cfg.depth, cudaMemcpyDeviceToHost, st));
    QVTS_CUDA(cudaMemcpyAsync(ctr, m.counters.p, sizeof(ctr), cudaMemcpyDeviceToHost, st));
    QVTS_CUDA(cudaStreamSynchronize(st));
    QVTS_CUDA(cudaEventRecord(m.pg_join, st));
    QVTS_CUDA(cudaStreamWaitEvent(cst, m.pg_join, 0));
    for (int d = 0; d < cfg.depth; ++d) {
        nv[d] = cnt[d]; m.vl[d].n = cnt[d]; m.ql[d].nwork = cnt[d];
        m.ql[d].mapped = false; m.ql[d].vmap_ptr = nullptr;    // the graph's levels are unmapped
    }
    nv[cfg.depth] = (long long)ctr[1];
    m.last_flagged = (long long)ctr[0];
    m.last_skipped = (long long)(ctr[2] + ctr[3]);
    m.last_xdraws = false;
    m.last_depth = cfg.depth;
    m.last_shard_level = -1;
    m.last_n = cfg.n_samples;
    m.last_trace = false;
    return QVTS_OK;
}

qvts_status plan_levels(Model &m, const RootBatch &roots, const qvts_plan_cfg &cfg, const qvts_comm *comm,
                        cudaStream_t st, long long *nv_out) {
    qvts_status s = QVTS_ERR_INVALID_ARG;
#define QVTS_PLAN(MASK) s = plan_levels_t<MASK>(m, roots, cfg, comm, st, nv_out)
    QVTS_DISPATCH_MASK(m.mask, QVTS_PLAN);
#undef QVTS_PLAN
    return s;
}

}  // namespace qvts

using namespace qvts;

extern "C" qvts_status qvts_plan_step(qvts_model *m, const float *root_dev, const qvts_plan_cfg *cfg,
                                      const qvts_comm *comm, qvts_plan_result *res, void *stream) {
    qvts::NvtxRange nvtx_range__("qvts_plan_step");
    if (!m || !root_dev || !cfg || !res) { set_error("NULL argument"); return QVTS_ERR_INVALID_ARG; }
    if (cfg->depth < 1 || cfg->depth > 8 || cfg->n_samples < 1 || cfg->n_samples > 4096) {
        set_error("depth must be 1..8 and n_samples 1..4096"); return QVTS_ERR_INVALID_ARG;
    }
    if (comm && (comm->nranks < 1 || comm->rank < 0 || comm->rank >= comm->nranks ||
                 (comm->nranks > 1 && !comm->allreduce_sum_f64))) {
        set_error("bad comm"); return QVTS_ERR_INVALID_ARG;
    }
    if (!m->have_q) { set_error("run qvts_value_iteration before planning"); return QVTS_ERR_STATE; }
    if (cfg->leaf_bound != QVTS_LEAF_QMDP && cfg->leaf_bound != QVTS_LEAF_FIB) { set_error("bad leaf_bound"); return QVTS_ERR_INVALID_ARG; }
    if (cfg->leaf_bound == QVTS_LEAF_FIB && !m->have_fib) { set_error("run qvts_fib_iteration before FIB leaves"); return QVTS_ERR_STATE; }
    if (cfg->sampler != QVTS_SAMPLER_MARGINAL && cfg->sampler != QVTS_SAMPLER_ANCESTRAL) { set_error("bad sampler"); return QVTS_ERR_INVALID_ARG; }
    QVTS_CUDA(cudaSetDevice(m->device));
    cudaStream_t st = (cudaStream_t)stream;
    QVTS_TRY(m->ep_root_step.ensure(sizeof(uint32_t) * 2));
    QVTS_TRY(m->ep_root_ep.ensure(sizeof(uint32_t) * 2));
    uint32_t keys[2] = {cfg->step, cfg->episode};
    QVTS_CUDA(cudaMemcpyAsync(m->ep_root_step.p, &keys[0], sizeof(uint32_t), cudaMemcpyHostToDevice, st));
    QVTS_CUDA(cudaMemcpyAsync(m->ep_root_ep.p, &keys[1], sizeof(uint32_t), cudaMemcpyHostToDevice, st));
    RootBatch rb{root_dev, (long long)m->HW, 1, m->ep_root_step.as<uint32_t>(), m->ep_root_ep.as<uint32_t>()};
    long long nv[kMaxLevels + 1] = {0};
    double q[9];
    // small single-GPU trees: the graph-captured step (QVTS_PLAN_GRAPH=0 keeps the level-synchronous one)
    long long vmax[kMaxLevels + 1];
    const char *ev_graph = std::getenv("QVTS_PLAN_GRAPH");
    const bool use_graph = (!ev_graph || std::atoi(ev_graph) != 0) && (!comm || comm->nranks == 1) &&
                           !cfg->want_trace && !m->prof && graph_eligible(*m, *cfg, vmax);
    if (use_graph) {
        QVTS_TRY(plan_step_graph(*m, root_dev, *cfg, vmax, st, q, nv));
    } else {
        QVTS_CUDA(cudaEventRecord(m->ev0, st));
        QVTS_TRY(plan_levels(*m, rb, *cfg, comm, st, nv));
        QVTS_CUDA(cudaEventRecord(m->ev1, st));
        QVTS_CUDA(cudaMemcpyAsync(q, m->ql[0].Q.p, sizeof(double) * m->NA, cudaMemcpyDeviceToHost, st));
        QVTS_CUDA(cudaStreamSynchronize(st));
    }
    float ms = 0.f;
    QVTS_CUDA(cudaEventElapsedTime(&ms, m->ev0, m->ev1));
    prof_collect(*m);
    std::memset(res, 0, sizeof(*res));
    res->shard_level = m->last_shard_level;
    res->n_actions = m->NA;
    int arg = 0;
    for (int j = 0; j < m->NA; ++j) {
        res->q_root[j] = q[j];
        if (q[j] > q[arg]) arg = j;    // ties -> lowest stencil id (R16)
    }
    res->action = m->action_id[arg];
    long long tot = 0;
    for (int d = 0; d <= cfg->depth; ++d) {
        res->n_vnodes[d] = nv[d];
        if (d) tot += nv[d];
    }
    res->n_belief_updates = tot;
    res->device_ms = ms;
    res->n_flag_candidates = m->last_flagged;
    res->n_tiles_skipped = m->last_skipped;
    return QVTS_OK;
}

extern "C" qvts_status qvts_belief_update(qvts_model *m, const float *b_dev, int32_t action, int32_t z,
                                          float *out_dev, double *p_obs_out, void *stream) {
    qvts::NvtxRange nvtx_range__("qvts_belief_update");
    if (!m || !b_dev || !out_dev) { set_error("NULL argument"); return QVTS_ERR_INVALID_ARG; }
    // one (b, a, z): the batched kernels with n = 1 (selected-z normaliser, then the correction)
    return qvts_belief_update_batch(m, b_dev, m->HW, 1, &action, &z, out_dev, m->HW, p_obs_out, stream);
}

// Batched Eq. 3, pass 1: M_g[s] = sum over class-s cells of bbar_{a_g}(y) for the selected action
// only (correct_predict's 4-cell groups, k_correct's tiling), one fp64 partial per (belief, tile,
// class); pass 2 (k_bu_p) sums the tiles in order and forms P(z|b,a) = sum_s O[s][z] M[s].
template <uint32_t MASK>
// Eq. 3's normaliser for the one selected (a, z) of each belief, per row tile:
// part[g][tile] = sum_y O[sig(y)][z] bbar_a(y) (fp64 per thread, fixed-order block reduction).
// Only P(z | b, a) at the selected z is needed (k_correct's weights and the caller's p_obs).
__global__ void __launch_bounds__(256) k_bu_marg(CorrectArgs a, double *__restrict__ part) {
    constexpr int NA = mask_count(MASK);
    const long long grp = blockIdx.x / a.ntiles;
    const int tile = blockIdx.x % a.ntiles;
    const long long q = a.sel_q[grp];
    const int j = (int)(q % NA), k = action_of<MASK>(j);
    const float *__restrict__ b = a.beliefs + (q / NA) * a.bstride;
    const int W = a.W;
    const bool vec = a.vec_in != 0;                 // set on the host (alignment of b included)
    __shared__ float s_o[16];                       // O[s][z] of the selected z
    if (threadIdx.x < 16) s_o[threadIdx.x] = (float)a.O64[threadIdx.x * 16 + a.sel_z[grp]];
    __syncthreads();
    double acc = 0.0;
    const int r_end = min(a.H, (tile + 1) * a.rows_cta);
    for (int idx = threadIdx.x; idx < a.rows_cta * a.G; idx += 256) {
        const int r = tile * a.rows_cta + idx / a.G, c0 = 4 * (idx % a.G);
        if (r >= r_end) break;
        float nbh[3][6];
#pragma unroll
        for (int dr = 0; dr < 3; ++dr) {
            const int rr = r + dr - 1;
            const bool rok = rr >= 0 && rr < a.H;
            const float *row = b + (long long)rr * W;
            if (vec) {
                const float4 m4 = rok ? __ldg(reinterpret_cast<const float4 *>(row + c0)) : make_float4(0.f, 0.f, 0.f, 0.f);
                nbh[dr][0] = (rok && c0 > 0) ? __ldg(row + c0 - 1) : 0.f;
                nbh[dr][1] = m4.x; nbh[dr][2] = m4.y; nbh[dr][3] = m4.z; nbh[dr][4] = m4.w;
                nbh[dr][5] = (rok && c0 + 4 < W) ? __ldg(row + c0 + 4) : 0.f;
            } else {
#pragma unroll
                for (int i = 0; i < 6; ++i) {
                    const int cc = c0 - 1 + i;
                    nbh[dr][i] = (rok && cc >= 0 && cc < W) ? __ldg(row + cc) : 0.f;
                }
            }
        }
        float bb[4];
        int sg[4];
        switch (k) {
            case 0: correct_predict<0>(a, r, c0, nbh, bb, sg); break;
            case 1: correct_predict<1>(a, r, c0, nbh, bb, sg); break;
            case 2: correct_predict<2>(a, r, c0, nbh, bb, sg); break;
            case 3: correct_predict<3>(a, r, c0, nbh, bb, sg); break;
            case 4: correct_predict<4>(a, r, c0, nbh, bb, sg); break;
            case 5: correct_predict<5>(a, r, c0, nbh, bb, sg); break;
            case 6: correct_predict<6>(a, r, c0, nbh, bb, sg); break;
            case 7: correct_predict<7>(a, r, c0, nbh, bb, sg); break;
            default: correct_predict<8>(a, r, c0, nbh, bb, sg); break;
        }
#pragma unroll
        for (int i = 0; i < 4; ++i) acc += (double)(s_o[sg[i]] * bb[i]);
    }
    // fixed-order reduction: butterfly within each warp, then the 8 warp sums in warp order
    __shared__ double wsum[8];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) wsum[warp] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
        double sm = 0.0;
#pragma unroll
        for (int w2 = 0; w2 < 8; ++w2) sm += wsum[w2];
        part[grp * a.ntiles + tile] = sm;
    }
}
// Batched Eq. 3 in ONE pass over b (K9 at HBM rate): one thread-block cluster of NC CTAs per
// belief, CTA rank r owns rows [r R, (r+1) R).  Each CTA stages its rows (+1-row halo) in shared
// memory with one cp.async burst; every thread predicts its <= G groups of 4 cells ONCE, keeps
// O[sig(y)][z] bbar_a(y) in registers and adds its part of P(z|b,a) = sum_y O[sig(y)][z] bbar_a(y)
// (fp32 per thread, fp64 across threads in fixed order); the cluster sums the NC parts in rank
// order through DSMEM (every CTA gets the same bits) and the thread writes
// b' = (O[sig][z] bbar) (1/P) from its registers with streaming float4 stores: b is read once and
// b' written once.
//
// Per cell the prediction is bbar = p_int b(y - d_a) + p_lat (b(y - d_l1) + b(y - d_l2)) +
// c(m8(y)) b(y), c = p_stay + p_int [y + d_a blocked] + p_lat ([y + d_l1 blocked] +
// [y + d_l2 blocked]) (the blocked moves' mass stays, Eq. 2), with c tabulated over the 256
// occupancy bytes and O[sig][z] over the 32 (occupied, sig) codes (0 for an occupied cell) once
// per CTA: three tap loads, two table loads and five FP operations per cell.  One code path for
// every action: the three source taps (the intended move and its two ring laterals, reading R3)
// are runtime offsets into the staged rows; stay has coefficients (1, 0, 0).  The fp32 rounding
// differs from k_correct's by O(1 ulp) (the two-pass path, compared in the tests).
struct BuActs { int act[9]; };
struct BuArgs {
    const float *beliefs;
    long long bstride;
    const uint8_t *m8, *cell;
    const double *O64;
    const int32_t *sel_q, *sel_z, *sel_out;
    float *out;
    long long ostride;
    double *pout;
    int n, NA, H, W, rows, TPc;
    float p_int, p_stay, p_lat;
    BuActs acts;
};
constexpr int kBuThreads = 256;
constexpr int kBuGroups = 8;         // 4-cell groups per thread: rows * W / 4 <= 8 * 256

__global__ void __launch_bounds__(kBuThreads, 4) k_bu_cluster(BuArgs a) {
    namespace cg = cooperative_groups;
    constexpr int G = kBuGroups;
    cg::cluster_group cl = cg::this_cluster();
    const int NC = (int)cl.num_blocks();
    const int rank = (int)cl.block_rank();
    const long long g = blockIdx.x / NC;
    const long long q = a.sel_q[g];
    const int zsel = a.sel_z[g];
    const int k = a.acts.act[q % a.NA];
    const float *__restrict__ b = a.beliefs + (q / a.NA) * a.bstride;
    const int W = a.W, TPc = a.TPc, W4 = W >> 2;
    const int r0 = rank * a.rows, r1 = min(a.H, r0 + a.rows), nrows = r1 - r0;
    const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
    extern __shared__ float4 bu_smem4[];
    float *stile = reinterpret_cast<float *>(bu_smem4);
    __shared__ float s_c[256], s_t[32];
    __shared__ double wsum[8], s_parts[8];        // s_parts[r]: rank r's part, pushed by rank r
    // stage rows [r0 - 1, r1 + 1) by bulk (TMA) copies, one row per lane of warp 0, completion on
    // an mbarrier; off-map rows and the halo columns are zeroed by the other threads meanwhile
    const int nr = nrows + 2;
    __shared__ alignas(8) unsigned long long s_bar;
    __shared__ alignas(8) unsigned long long s_rbar;   // NC arrivals: every rank's part is here
    const uint32_t bar = (uint32_t)__cvta_generic_to_shared(&s_bar);
    const uint32_t rbar = (uint32_t)__cvta_generic_to_shared(&s_rbar);
    const int lo = r0 == 0 ? 1 : 0, hi = r1 == a.H ? nr - 1 : nr;     // on-map staged rows
    if (t == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(bar));
        asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(rbar), "r"(NC));
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(bar),
                     "r"((uint32_t)((hi - lo) * W * 4)) : "memory");
    }
    // every CTA's barriers are initialised before any rank pushes into them: arrive now, wait
    // just before the push (the staging and the prediction run in between)
    asm volatile("barrier.cluster.arrive.relaxed.aligned;\n" ::: "memory");
    if (warp == 0) {
        __syncwarp();
        for (int tr = lo + lane; tr < hi; tr += 32)
            asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                             (uint32_t)__cvta_generic_to_shared(stile + tr * TPc + 4)),
                         "l"(b + (long long)(r0 - 1 + tr) * W), "r"((uint32_t)(W * 4)), "r"(bar)
                         : "memory");
    } else {
        for (int tr = t - 32; tr < nr; tr += kBuThreads - 32) {
            stile[tr * TPc + 3] = 0.f;
            stile[tr * TPc + 4 + W] = 0.f;
        }
        for (int c = t - 32; c < W; c += kBuThreads - 32) {
            if (lo) stile[4 + c] = 0.f;
            if (hi < nr) stile[(nr - 1) * TPc + 4 + c] = 0.f;
        }
    }
    // meanwhile: this action's staying-mass coefficient over the occupancy bytes, the O weights
    const bool stay = k == 4;
    const int k1 = stay ? 4 : lat1_rt(k), k2 = stay ? 4 : lat2_rt(k);
    {
        float c = stay ? 1.f : a.p_stay;
        if (!stay) {
            if ((t >> nbit(k)) & 1) c += a.p_int;
            if ((t >> nbit(k1)) & 1) c += a.p_lat;
            if ((t >> nbit(k2)) & 1) c += a.p_lat;
        }
        s_c[t] = c;
        if (t < 32) s_t[t] = t < 16 ? (float)a.O64[t * 16 + zsel] : 0.f;
    }
    const int offa = -st_dr(k) * TPc - st_dc(k), off1 = -st_dr(k1) * TPc - st_dc(k1), off2 = -st_dr(k2) * TPc - st_dc(k2);
    const float c_int = stay ? 0.f : a.p_int, c_lat = stay ? 0.f : a.p_lat;
    // a thread owns one 4-cell column group and every RPP-th row of the CTA (W / 4 divides 256,
    // checked on the host), so all addresses advance by constants
    const int RPP = kBuThreads / W4, c0 = 4 * (t % W4), rl0 = t / W4;
    const unsigned int *cellp = reinterpret_cast<const unsigned int *>(a.cell + (long long)(r0 + rl0) * W + c0);
    const unsigned int *m8p = reinterpret_cast<const unsigned int *>(a.m8 + (long long)(r0 + rl0) * W + c0);
    uint32_t info4[G], m84[G];
#pragma unroll
    for (int gg = 0; gg < G; ++gg) {
        info4[gg] = 0u;
        m84[gg] = 0u;
        if (rl0 + RPP * gg < nrows) {
            info4[gg] = __ldg(cellp + gg * (RPP * W4));
            m84[gg] = __ldg(m8p + gg * (RPP * W4));
        }
    }
    __syncthreads();                             // tables and zeros visible
    asm volatile(
        "{\n .reg .pred P1;\n WAIT_%=:\n"
        " mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n"
        " @!P1 bra WAIT_%=;\n}\n" ::"r"(bar) : "memory");
    const float *rowp = stile + (rl0 + 1) * TPc + 4 + c0;
    float ob[G][4];                              // O[sig][z] bbar of the thread's cells
    float accf = 0.f;
#pragma unroll
    for (int gg = 0; gg < G; ++gg) {
#pragma unroll
        for (int i = 0; i < 4; ++i) ob[gg][i] = 0.f;
        if (rl0 + RPP * gg < nrows) {
            const float4 b4 = *reinterpret_cast<const float4 *>(rowp);
            const float b0v[4] = {b4.x, b4.y, b4.z, b4.w};
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const float sa = rowp[offa + i], s1 = rowp[off1 + i], s2 = rowp[off2 + i];
                const float cs = s_c[(m84[gg] >> (8 * i)) & 255u];
                const float v = fmaf(c_lat, s1 + s2, fmaf(c_int, sa, cs * b0v[i]));
                ob[gg][i] = s_t[(info4[gg] >> (8 * i)) & 31u] * v;        // occupied: 0
                accf += ob[gg][i];
            }
        }
        rowp += RPP * TPc;
    }
    // fixed-order reduction: fp64 butterfly within each warp, then the 8 warp sums in order
    double acc = (double)accf;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) wsum[warp] = acc;
    __syncthreads();
    // push this rank's part into slot [rank] of every CTA of the cluster (thread rr -> rank rr) and
    // arrive on that CTA's barrier (release: the store is visible with the arrival); then wait for
    // the NC parts here and sum them in rank order -- the same bits on every CTA.  A CTA leaves only
    // after all NC arrivals on its own barrier, so no rank writes into an exited CTA.
    asm volatile("barrier.cluster.wait.aligned;\n" ::: "memory");
    if (t < NC) {
        double part = 0.0;
#pragma unroll
        for (int w2 = 0; w2 < 8; ++w2) part += wsum[w2];
        uint32_t rp, rb;
        asm volatile("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(rp) : "r"((uint32_t)__cvta_generic_to_shared(&s_parts[rank])), "r"(t));
        asm volatile("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(rb) : "r"(rbar), "r"(t));
        asm volatile("st.shared::cluster.f64 [%0], %1;\n" ::"r"(rp), "d"(part) : "memory");
        asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];\n" ::"r"(rb) : "memory");
    }
    asm volatile(
        "{\n .reg .pred P1;\n WAIT_%=:\n"
        " mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 P1, [%0], 0;\n"
        " @!P1 bra WAIT_%=;\n}\n" ::"r"(rbar) : "memory");
    double P = 0.0;
    for (int rr = 0; rr < NC; ++rr) P += s_parts[rr];
    // a zero-likelihood z writes zeros (the host reports QVTS_ERR_ZERO_LIKELIHOOD)
    const float inv = P > 1e-30 ? (float)(1.0 / P) : 0.f;
    if (t == 0 && rank == 0) a.pout[g] = P;
    float *outp = a.out + (long long)a.sel_out[g] * a.ostride + (long long)(r0 + rl0) * W + c0;
#pragma unroll
    for (int gg = 0; gg < G; ++gg) {
        if (rl0 + RPP * gg < nrows)
            __stcs(reinterpret_cast<float4 *>(outp),
                   make_float4(ob[gg][0] * inv, ob[gg][1] * inv, ob[gg][2] * inv, ob[gg][3] * inv));
        outp += RPP * W;
    }
}

// P(z | b, a) of each selected pair: the tile partials summed in order, into the Q-node layout
// k_correct reads (P[q][z]) and the caller's per-belief array
__global__ void k_bu_p(const double *__restrict__ part, int ntiles, const int32_t *__restrict__ sel_q,
                       const int32_t *__restrict__ sel_z, int n, double *__restrict__ P, double *__restrict__ pout) {
    const int g = blockIdx.x * blockDim.x + threadIdx.x;
    if (g >= n) return;
    double pz = 0.0;
    for (int t2 = 0; t2 < ntiles; ++t2) pz += part[(long long)g * ntiles + t2];
    P[(long long)sel_q[g] * 16 + sel_z[g]] = pz;
    pout[g] = pz;
}

extern "C" qvts_status qvts_belief_update_batch(qvts_model *m, const float *b_dev, int64_t b_stride, int32_t n,
                                                const int32_t *actions, const int32_t *zs, float *out_dev,
                                                int64_t out_stride, double *p_obs_out, void *stream) {
    qvts::NvtxRange nvtx_range__("qvts_belief_update_batch");
    if (!m || (n > 0 && (!b_dev || !actions || !zs || !out_dev))) { set_error("NULL argument"); return QVTS_ERR_INVALID_ARG; }
    if (n < 0 || b_stride < m->HW || out_stride < m->HW) { set_error("bad n or stride"); return QVTS_ERR_INVALID_ARG; }
    if (n == 0) return QVTS_OK;
    QVTS_CUDA(cudaSetDevice(m->device));
    cudaStream_t st = (cudaStream_t)stream;
    const int NA = m->NA;
    // the selection (Q-node, z, output slot) of every pair through page-locked staging: a true
    // async upload, and P's readback below the same way
    QVTS_TRY(m->bu_host.ensure(sizeof(int32_t) * 3 * (size_t)n + sizeof(double) * (size_t)n + 16));
    int32_t *sel = m->bu_host.as<int32_t>();
    double *p_host = reinterpret_cast<double *>(m->bu_host.as<char>() + ((sizeof(int32_t) * 3 * (size_t)n + 15) & ~(size_t)15));
    int lut[9];                                  // stencil id -> action index (-1: not in the set)
    for (int k = 0; k < 9; ++k) lut[k] = -1;
    for (int i = 0; i < NA; ++i) lut[m->action_id[i]] = i;
    for (int g = 0; g < n; ++g) {
        const int j = (actions[g] >= 0 && actions[g] < 9) ? lut[actions[g]] : -1;
        if (j < 0 || zs[g] < 0 || zs[g] > 15) { set_error("action not in the action set or z out of range"); return QVTS_ERR_INVALID_ARG; }
        sel[g] = g * NA + j;
        sel[n + g] = zs[g];
        sel[2 * n + g] = g;
    }
    QVTS_TRY(m->bu_off.ensure(sizeof(int32_t) * 3 * (size_t)n));
    QVTS_TRY(m->bu_P.ensure(sizeof(double) * (size_t)n));
    QVTS_CUDA(cudaMemcpyAsync(m->bu_off.p, sel, sizeof(int32_t) * 3 * (size_t)n, cudaMemcpyHostToDevice, st));
    const int32_t *d_sel = m->bu_off.as<int32_t>();
    auto finish = [&]() -> qvts_status {
        QVTS_CUDA(cudaMemcpyAsync(p_host, m->bu_P.p, sizeof(double) * n, cudaMemcpyDeviceToHost, st));
        QVTS_CUDA(cudaStreamSynchronize(st));
        bool zero = false;
        for (int g = 0; g < n; ++g) {
            if (p_obs_out) p_obs_out[g] = p_host[g];
            if (!(p_host[g] > 1e-30)) zero = true;
        }
        if (zero) { set_error("zero-likelihood observation in the batch"); return QVTS_ERR_ZERO_LIKELIHOOD; }
        return QVTS_OK;
    };
    // one pass per belief on a thread-block cluster when the rows fit: 16-byte rows, W / 4 dividing
    // 256 (the column-group mapping), a cluster of NC <= 8 CTAs whose rows take <= kBuGroups
    // groups of 4 cells per thread; otherwise the two-pass path (normaliser, then k_correct)
    {
        const bool vec = (m->W & 3) == 0 && (b_stride & 3) == 0 && (out_stride & 3) == 0 &&
                         (reinterpret_cast<uintptr_t>(b_dev) & 15) == 0 && (reinterpret_cast<uintptr_t>(out_dev) & 15) == 0;
        const int W4 = m->W / 4, tp = m->W + 8;
        const bool groups_ok = W4 >= 1 && 256 % W4 == 0;
        // the smallest cluster (<= 8 CTAs, portable) whose rows fit kBuGroups groups per thread;
        // 16-CTA clusters of 16 rows (non-portable, 6 CTAs per SM) measured slower: 0.50 vs 0.42 ms
        int NC = 0, rows = 0;
        for (int nc = 1; nc <= 8 && groups_ok && !NC; ++nc) {
            const int r = (m->H + nc - 1) / nc;
            if ((long long)r * W4 <= (long long)kBuGroups * kBuThreads) { NC = nc; rows = r; }
        }
        const char *ev_bu = std::getenv("QVTS_BU_CLUSTER");          // read per call (0: two-pass path)
        if (vec && NC > 0 && (!ev_bu || std::atoi(ev_bu) != 0) && (long long)n * NC <= 0x7FFFFFFFLL) {
            BuArgs ba;
            ba.beliefs = b_dev; ba.bstride = b_stride; ba.m8 = m->d_m8.as<uint8_t>(); ba.cell = m->d_cell.as<uint8_t>();
            ba.O64 = m->d_O64.as<double>(); ba.sel_q = d_sel; ba.sel_z = d_sel + n; ba.sel_out = d_sel + 2 * n;
            ba.out = out_dev; ba.ostride = out_stride; ba.pout = m->bu_P.as<double>();
            ba.n = n; ba.NA = NA; ba.H = m->H; ba.W = m->W; ba.rows = rows; ba.TPc = tp;
            ba.p_int = (float)m->p_int; ba.p_stay = (float)m->p_stay; ba.p_lat = (float)m->p_lat;
            for (int j = 0; j < 9; ++j) ba.acts.act[j] = j < NA ? m->action_id[j] : 4;
            const size_t smem = sizeof(float) * (size_t)(rows + 2) * tp;
            auto kfn = k_bu_cluster;
            QVTS_CUDA(cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
            cudaLaunchConfig_t lc = {};
            lc.gridDim = dim3((unsigned)(n * NC));
            lc.blockDim = dim3(kBuThreads);
            lc.dynamicSmemBytes = smem;
            lc.stream = st;
            cudaLaunchAttribute attr[1];
            attr[0].id = cudaLaunchAttributeClusterDimension;
            attr[0].val.clusterDim.x = NC;
            attr[0].val.clusterDim.y = 1;
            attr[0].val.clusterDim.z = 1;
            lc.attrs = attr;
            lc.numAttrs = 1;
            QVTS_CUDA(cudaLaunchKernelEx(&lc, kfn, ba));
            QVTS_CUDA(cudaGetLastError());
            return finish();
        }
    }
    CorrectArgs c;
    std::memset(&c, 0, sizeof(c));
    c.beliefs = b_dev; c.bstride = b_stride; c.m8 = m->d_m8.as<uint8_t>(); c.cell = m->d_cell.as<uint8_t>();
    c.O64 = m->d_O64.as<double>(); c.H = m->H; c.W = m->W; c.G = (m->W + 3) / 4;
    // CTAs of ~BU_GROUPS groups of 4 cells (the plan's 1024 leave the one-child case latency-bound)
    const char *ev_groups = std::getenv("QVTS_BU_GROUPS");     // read per call
    const int bu_groups = ev_groups ? std::max(256, std::atoi(ev_groups)) : 2048;   // 32-row tiles at W = 256
    c.rows_cta = std::min(m->H, std::max(1, bu_groups / std::max(1, c.G)));
    c.ntiles = (m->H + c.rows_cta - 1) / c.rows_cta;
    c.p_int = (float)m->p_int; c.p_stay = (float)m->p_stay; c.p_lat = (float)m->p_lat; c.qsel = -1;
    c.sel_q = d_sel; c.sel_z = d_sel + n; c.sel_out = d_sel + 2 * n;
    c.child = out_dev; c.cstride = out_stride;
    QVTS_TRY(m->part.ensure(sizeof(double) * (size_t)n * c.ntiles));
    QVTS_TRY(m->bu_R.ensure(sizeof(double) * (size_t)n * NA * 16));     // P in the Q-node layout
    c.P = m->bu_R.as<double>();
    const long long nblocks = (long long)n * c.ntiles;
    if (nblocks > 0x7FFFFFFFLL) { set_error("batch too large"); return QVTS_ERR_INVALID_ARG; }
#define QVTS_BUB(MASK)                                                                                          \
    {                                                                                                           \
        correct_stage(c);                                                                                       \
        k_bu_marg<MASK><<<(unsigned)nblocks, 256, 0, st>>>(c, m->part.as<double>());                            \
        k_bu_p<<<nblk(n, 256), 256, 0, st>>>(m->part.as<double>(), c.ntiles, d_sel, d_sel + n, n,               \
                                             m->bu_R.as<double>(), m->bu_P.as<double>());                        \
        { const size_t csm_ = correct_stage(c); \
        k_correct<MASK><<<(unsigned)nblocks, 256, csm_, st>>>(c); } \
    }
    QVTS_DISPATCH_MASK(m->mask, QVTS_BUB);
#undef QVTS_BUB
    QVTS_CUDA(cudaGetLastError());
    return finish();
}

// ---- trace accessors ----------------------------------------------------------------------------
static qvts_status check_level(const qvts_model *m, int level, bool qlevel) {
    if (!m) { set_error("model is NULL"); return QVTS_ERR_INVALID_ARG; }
    if (m->last_depth < 0) { set_error("no plan step has run"); return QVTS_ERR_STATE; }
    if (level < 0 || level > m->last_depth - (qlevel ? 1 : 0)) { set_error("level out of range"); return QVTS_ERR_INVALID_ARG; }
    return QVTS_OK;
}

template <class T>
static qvts_status d2h(T *dst, const DevBuf &b, size_t count) {
    if (!dst || count == 0) return QVTS_OK;
    QVTS_CUDA(cudaMemcpy(dst, b.p, sizeof(T) * count, cudaMemcpyDeviceToHost));
    return QVTS_OK;
}

extern "C" qvts_status qvts_trace_qnodes(const qvts_model *m, int32_t level, uint64_t *path, double *R, double *P,
                                         uint16_t *cnt, double *Q, uint8_t *z) {
    QVTS_TRY(check_level(m, level, true));
    QVTS_CUDA(cudaSetDevice(m->device));
    const QLevel &ql = m->ql[level];
    const long long nq = ql.nwork * m->NA;
    if (path) {
        // Q-node path = parent V-node path | (a+1) << 8*level
        std::vector<uint64_t> vp(m->vl[level].n);
        std::vector<int32_t> vmap;
        QVTS_TRY(d2h(vp.data(), m->vl[level].path, vp.size()));
        if (ql.mapped) {
            vmap.resize(ql.nwork);
            if (!vmap.empty()) QVTS_CUDA(cudaMemcpy(vmap.data(), ql.vmap_ptr, sizeof(int32_t) * vmap.size(), cudaMemcpyDeviceToHost));
        }
        for (long long q = 0; q < nq; ++q) {
            const long long w = q / m->NA;
            const long long v = ql.mapped ? vmap[w] : w;
            path[q] = vp[v] | ((uint64_t)(m->action_id[q % m->NA] + 1) << (8 * level));
        }
    }
    QVTS_TRY(d2h(R, ql.R, nq));
    QVTS_TRY(d2h(P, ql.P, nq * 16));
    QVTS_TRY(d2h(cnt, ql.cnt, nq * 16));
    QVTS_TRY(d2h(Q, ql.Q, nq));
    if (z) {
        if (!m->last_trace) { set_error("draws need want_trace"); return QVTS_ERR_STATE; }
        QVTS_TRY(d2h(z, ql.zdraw, nq * m->last_n));
    }
    return QVTS_OK;
}

extern "C" qvts_status qvts_trace_vnodes(const qvts_model *m, int32_t level, uint64_t *path, int32_t *parent_q,
                                         int32_t *zobs, int32_t *freq, double *V) {
    QVTS_TRY(check_level(m, level, true));
    QVTS_CUDA(cudaSetDevice(m->device));
    const VLevel &vl = m->vl[level];
    QVTS_TRY(d2h(path, vl.path, vl.n));
    if (level > 0) {
        QVTS_TRY(d2h(parent_q, vl.parent_q, vl.n));
        QVTS_TRY(d2h(zobs, vl.z, vl.n));
        QVTS_TRY(d2h(freq, vl.f, vl.n));
    }
    QVTS_TRY(d2h(V, vl.V, vl.n));
    return QVTS_OK;
}

extern "C" qvts_status qvts_trace_leaf_values(const qvts_model *m, double *V) {
    if (!m || !V) { set_error("NULL argument"); return QVTS_ERR_INVALID_ARG; }
    if (m->last_depth < 0 || !m->last_trace) { set_error("needs a plan step with want_trace"); return QVTS_ERR_STATE; }
    QVTS_CUDA(cudaSetDevice(m->device));
    const QLevel &ql = m->ql[m->last_depth - 1];
    return d2h(V, ql.leafV, ql.nwork * m->NA * 16);
}

extern "C" qvts_status qvts_trace_belief(const qvts_model *m, int32_t level, int64_t index, float *out_host) {
    QVTS_TRY(check_level(m, level, true));
    if (level == 0) { set_error("the root belief is the caller's buffer"); return QVTS_ERR_INVALID_ARG; }
    if (index < 0 || index >= m->vl[level].n || !out_host) { set_error("index out of range"); return QVTS_ERR_INVALID_ARG; }
    QVTS_CUDA(cudaSetDevice(m->device));
    QVTS_CUDA(cudaMemcpy(out_host, m->vl[level].belief.as<float>() + (size_t)index * m->HWp, sizeof(float) * m->HW,
                         cudaMemcpyDeviceToHost));
    return QVTS_OK;
}

// Number of V-nodes per level of the last plan step (levels 0..depth) — convenience for bindings.
extern "C" qvts_status qvts_trace_state_draws(const qvts_model *m, int32_t level, int32_t *x) {
    QVTS_TRY(check_level(m, level, true));
    if (!x) { set_error("NULL argument"); return QVTS_ERR_INVALID_ARG; }
    if (!m->last_xdraws) { set_error("state draws need want_trace and the ancestral sampler"); return QVTS_ERR_STATE; }
    QVTS_CUDA(cudaSetDevice(m->device));
    const QLevel &ql = m->ql[level];
    return d2h(x, ql.xdraw, (size_t)ql.nwork * m->NA * m->last_n);
}

extern "C" qvts_status qvts_trace_counts(const qvts_model *m, int32_t *depth, int64_t *n_v, int64_t *n_qwork) {
    if (!m) { set_error("model is NULL"); return QVTS_ERR_INVALID_ARG; }
    if (m->last_depth < 0) { set_error("no plan step has run"); return QVTS_ERR_STATE; }
    if (depth) *depth = m->last_depth;
    for (int d = 0; d <= m->last_depth; ++d) {
        if (n_v) n_v[d] = d < m->last_depth ? m->vl[d].n : -1;
        if (n_qwork && d < m->last_depth) n_qwork[d] = m->ql[d].nwork;
    }
    return QVTS_OK;
}
