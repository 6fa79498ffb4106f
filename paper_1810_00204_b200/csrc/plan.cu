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
#include <cstring>

#include "qvts_internal.cuh"
#include "stencil.cuh"

namespace qvts {

// ---- Philox4x32-10 (Salmon et al. 2011) ---------------------------------
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

template <uint32_t MASK>
__device__ __forceinline__ int action_of(int j) {
    constexpr int NA = mask_count(MASK);
    int k = 0;
#pragma unroll
    for (int i = 0; i < NA; ++i)
        if (i == j) k = mask_action(MASK, i);
    return k;
}

// ---- S1 + S2 (+ S5): signature-binned histograms ----------------------------------------------
struct HistArgs {
    const float *beliefs;
    long long bstride;
    const int32_t *vmap;
    const BandInfo *bands;
    int nb;
    const uint32_t *entries;
    const float4 *qlist;
    const float *ctab;
    int H, W, TW, region_floats;
    float p_int, p_lat;
    double *part;
    int pstride;
};

template <uint32_t MASK, bool LEAF>
constexpr int hist_nv() {
    return mask_count(MASK) * (LEAF ? 1 + mask_count(MASK) : 1) + mask_count(MASK) + 1;
}

// One CTA = one (parent, band).  The band (+1-cell zero halo) is staged in shared memory; thread t
// walks its class-homogeneous slot stream, predicting bbar_a(y) for every action (gather form of
// the clamped stencil) and accumulating
//   M_a  += bbar_a(y)                   (bin = the thread's class sig(y); Eq. 3 normaliser)
//   Rp_a += c_a(y) b(y)                 (R(b,a) = (p_stay-1) sum b - sum c_a b + goal terms)
//   S_a,a' += bbar_a(y) Q'(y,a')        (LEAF only; Q' = Q - qbar)
// in fp32 registers, then reduces the per-thread values class by class in fixed order in fp64.
template <uint32_t MASK, bool LEAF>
__global__ void __launch_bounds__(kHistThreads) k_hist(HistArgs a) {
    constexpr int NA = mask_count(MASK);
    constexpr int NAP = (NA + 3) & ~3;
    constexpr int NV = hist_nv<MASK, LEAF>();
    constexpr int T = kHistThreads;
    extern __shared__ float4 smem4[];
    float *smem = reinterpret_cast<float *>(smem4);
    float *tile = smem;
    float *ctab = smem + a.region_floats;
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
    const int band = blockIdx.x % a.nb;
    const long long w = blockIdx.x / a.nb;
    const long long v = a.vmap ? (long long)a.vmap[w] : w;
    const BandInfo *bi = a.bands + band;
    const int row0 = bi->row0, nrows = bi->nrows, L = bi->L;
    const long long soff = bi->slot_off;
    const float *__restrict__ b = a.beliefs + v * a.bstride;
    const int TW = a.TW, TH = nrows + 2;

    for (int i = t; i < 256 * NAP; i += T) ctab[i] = a.ctab[i];
    for (int tr = warp; tr < TH; tr += T / 32) {
        const int r = row0 - 1 + tr;
        const bool rok = (r >= 0) && (r < a.H);
        const float *brow = b + (size_t)r * a.W;
        for (int tc = lane; tc < TW; tc += 32) {
            const int c = tc - 1;
            float val = 0.f;
            if (rok && c >= 0 && c < a.W) val = __ldg(brow + c);
            tile[tr * TW + tc] = val;
        }
    }
    __syncthreads();

    int off[9];
#pragma unroll
    for (int k = 0; k < 9; ++k) off[k] = st_dr(k) * TW + st_dc(k);

    float M[NA], Rp[NA], S[LEAF ? NA : 1][LEAF ? NA : 1];
    float mass = 0.f;
#pragma unroll
    for (int j = 0; j < NA; ++j) {
        M[j] = 0.f;
        Rp[j] = 0.f;
    }
    if (LEAF) {
#pragma unroll
        for (int j = 0; j < (LEAF ? NA : 1); ++j)
#pragma unroll
            for (int j2 = 0; j2 < (LEAF ? NA : 1); ++j2) S[j][j2] = 0.f;
    }
    const float p_int = a.p_int, p_lat = a.p_lat;

    for (int i = 0; i < L; ++i) {
        const long long slot = soff + (long long)i * T + t;
        const uint32_t e = __ldg(a.entries + slot);
        if (e == 0u) continue;
        const int ti = (int)(e & 0xFFFFu);
        const int m8 = (int)((e >> 16) & 0xFFu);
        float nb[9];
#pragma unroll
        for (int k = 0; k < 9; ++k) nb[k] = tile[ti + off[k]];
        float c[NAP];
        const float4 *c4 = reinterpret_cast<const float4 *>(ctab + m8 * NAP);
#pragma unroll
        for (int h = 0; h < NAP / 4; ++h) {
            const float4 cv = c4[h];
            c[4 * h] = cv.x; c[4 * h + 1] = cv.y; c[4 * h + 2] = cv.z; c[4 * h + 3] = cv.w;
        }
        float q[LEAF ? NAP : 1];
        if (LEAF) {
#pragma unroll
            for (int h = 0; h < (LEAF ? NAP / 4 : 0); ++h) {
                const float4 qv = __ldg(a.qlist + slot * (NAP / 4) + h);
                q[4 * h] = qv.x; q[4 * h + 1] = qv.y; q[4 * h + 2] = qv.z; q[4 * h + 3] = qv.w;
            }
        }
        const float b0 = nb[4];
        mass += b0;
#pragma unroll
        for (int j = 0; j < NA; ++j) {
            const int k = mask_action(MASK, j);
            float bb;
            if (k == 4) {
                bb = b0;
            } else {
                const float tt = c[j] * b0;
                Rp[j] += tt;
                bb = fmaf(p_int, nb[8 - k], tt);
                bb = fmaf(p_lat, nb[8 - lat1(k)] + nb[8 - lat2(k)], bb);
            }
            M[j] += bb;
            if (LEAF) {
#pragma unroll
                for (int j2 = 0; j2 < (LEAF ? NA : 1); ++j2) S[j][j2] = fmaf(bb, q[j2], S[j][j2]);
            }
        }
    }
    __syncthreads();   // the tile is dead; reuse the region for the reduction
    constexpr int RS = T + 1;   // padded row stride: no bank conflicts in the column sums
    float *red = smem;
#pragma unroll
    for (int j = 0; j < NA; ++j) red[j * RS + t] = M[j];
    if (LEAF) {
#pragma unroll
        for (int j = 0; j < (LEAF ? NA : 1); ++j)
#pragma unroll
            for (int j2 = 0; j2 < (LEAF ? NA : 1); ++j2) red[(NA + j * NA + j2) * RS + t] = S[j][j2];
    }
    constexpr int RPV = LEAF ? NA + NA * NA : NA;
#pragma unroll
    for (int j = 0; j < NA; ++j) red[(RPV + j) * RS + t] = Rp[j];
    red[(NV - 1) * RS + t] = mass;
    __syncthreads();
    constexpr int NCLS = 16 * RPV;       // class-binned outputs
    constexpr int NOUT = NCLS + NA + 1;
    double *dst = a.part + (w * a.nb + band) * (long long)a.pstride;
    for (int o = t; o < NOUT; o += T) {
        int vv, t0, t1;
        if (o < NCLS) {
            int cls;
            if (o < 16 * NA) { cls = o / NA; vv = o % NA; }
            else { const int r = o - 16 * NA; cls = r / (NA * NA); vv = NA + r % (NA * NA); }
            t0 = bi->cs[cls];
            t1 = bi->cs[cls + 1];
        } else {
            vv = RPV + (o - NCLS);
            t0 = 0;
            t1 = T;
        }
        double s = 0.0;
        for (int th = t0; th < t1; ++th) s += (double)red[vv * RS + th];
        dst[o] = s;
    }
}

// ---- S2 tail + S3 (+ S5 tail + S6 leaf backup): one warp per Q-node ---------------------------
struct ReduceArgs {
    const double *part;
    int pstride, nb;
    long long nq;
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
    const int32_t *gc_cell, *gc_act;
    const double *gc_val;
    int goal;
    double p_stay, gamma, qbar;
    double *R, *P;
    uint16_t *cnt, *umask;
    int32_t *U;
    uint8_t *zdraw;
    double *Q, *leafV;
    unsigned long long *nflag;
};

__device__ __forceinline__ double warp_sum_xor(double x) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
    return x;
}

template <uint32_t MASK, bool LEAF>
__global__ void __launch_bounds__(256) k_reduce(ReduceArgs a) {
    constexpr int NA = mask_count(MASK);
    const int lane = threadIdx.x & 31;
    const long long q = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
    if (q >= a.nq) return;
    const long long w = q / NA;
    const int j = (int)(q % NA);
    const int k = action_of<MASK>(j);
    const long long v = a.vmap ? (long long)a.vmap[w] : w;
    const double *pp = a.part + w * a.nb * (long long)a.pstride;
    constexpr int ROFF = LEAF ? 16 * NA * (1 + NA) : 16 * NA;

    double Ms = 0.0, tmp = 0.0;
    if (lane < 16)
        for (int bd = 0; bd < a.nb; ++bd) Ms += pp[(long long)bd * a.pstride + lane * NA + j];
    else if (lane == 16)
        for (int bd = 0; bd < a.nb; ++bd) tmp += pp[(long long)bd * a.pstride + ROFF + NA];
    else if (lane == 17)
        for (int bd = 0; bd < a.nb; ++bd) tmp += pp[(long long)bd * a.pstride + ROFF + j];
    const double mass = __shfl_sync(0xffffffffu, tmp, 16);
    const double Rp = __shfl_sync(0xffffffffu, tmp, 17);

    // R(b,a) = sum_x R(x,a) b(x) via the stencil identity of model.cu
    const float *bp = a.beliefs + v * a.bstride;
    double R = 0.0;
    if (lane == 0) {
        if (k == 4) {
            R = -2.0 * mass + 2.0 * (double)bp[a.goal];
        } else {
            R = (a.p_stay - 1.0) * mass - Rp;
            for (int g = 0; g < a.ngc; ++g)
                if (a.gc_act[g] == j) R += a.gc_val[g] * (double)bp[a.gc_cell[g]];
        }
    }
    // P(z|b,a) = sum_s O[s][z] M[s]   (Eq. 3 normaliser, fixed s order)
    double Pz = 0.0;
#pragma unroll
    for (int s = 0; s < 16; ++s) {
        const double m = __shfl_sync(0xffffffffu, Ms, s);
        if (lane < 16) Pz += a.O64[s * 16 + lane] * m;
    }
    double C[16];
    double acc = 0.0;
#pragma unroll
    for (int z = 0; z < 16; ++z) {
        acc += __shfl_sync(0xffffffffu, Pz, z);
        C[z] = acc;
    }
    // S3: n draws keyed by tree path (Appendix A.2-A.5)
    const uint64_t qpath = a.vpath[v] | ((uint64_t)(k + 1) << (8 * a.level));
    const int root = a.vroot[v];
    const uint32_t step = a.root_step[root], ep = a.root_ep[root];
    int cntk = 0, nflag = 0;
    for (int j0 = 0; j0 < a.n; j0 += 32) {
        const int jj = j0 + lane;
        const bool act = jj < a.n;
        int z = -1;
        if (act) {
            const uint4 r = philox4x32_10(make_uint4((uint32_t)jj, (uint32_t)qpath, (uint32_t)(qpath >> 32), step),
                                          make_uint2(a.seed, ep));
            const double u = ((double)(r.x >> 8) + 0.5) * (1.0 / 16777216.0);
            const double tt = u * C[15];
            z = 0;
            double gap = INFINITY;
#pragma unroll
            for (int kk = 0; kk < 16; ++kk) {
                z += (C[kk] <= tt) ? 1 : 0;
                if (kk < 15) gap = fmin(gap, fabs(tt - C[kk]));
            }
            z = min(z, 15);
            nflag += gap < 1e-6 ? 1 : 0;
            if (a.zdraw) a.zdraw[q * a.n + jj] = (uint8_t)z;
        }
#pragma unroll
        for (int kk = 0; kk < 16; ++kk) {
            const unsigned bal = __ballot_sync(0xffffffffu, z == kk);
            if (lane == kk) cntk += __popc(bal);
        }
    }
    const unsigned um = __ballot_sync(0xffffffffu, lane < 16 && cntk > 0) & 0xFFFFu;
    for (int o = 16; o > 0; o >>= 1) nflag += __shfl_xor_sync(0xffffffffu, nflag, o);
    if (lane < 16) {
        a.P[q * 16 + lane] = Pz;
        a.cnt[q * 16 + lane] = (uint16_t)cntk;
    }
    if (lane == 0) {
        a.R[q] = R;
        a.umask[q] = (uint16_t)um;
        a.U[q] = __popc(um);
        if (nflag && a.nflag) atomicAdd(a.nflag, (unsigned long long)nflag);
    }
    if (LEAF) {
        // S5: V(b') = qbar + max_a' [sum_s O[s][z] S[s][a']] / [sum_s O[s][z] M[s]]
        double Sv[LEAF ? NA : 1];
#pragma unroll
        for (int j2 = 0; j2 < (LEAF ? NA : 1); ++j2) Sv[j2] = 0.0;
        if (lane < 16)
            for (int bd = 0; bd < a.nb; ++bd) {
                const double *ps = pp + (long long)bd * a.pstride + 16 * NA + (lane * NA + j) * NA;
#pragma unroll
                for (int j2 = 0; j2 < (LEAF ? NA : 1); ++j2) Sv[j2] += ps[j2];
            }
        const double Rq = __shfl_sync(0xffffffffu, R, 0);
        double accq = 0.0;
        unsigned rem = um;
        while (rem) {
            const int z = __ffs(rem) - 1;
            rem &= rem - 1;
            const double Oz = lane < 16 ? a.O64[lane * 16 + z] : 0.0;
            const double Pzz = __shfl_sync(0xffffffffu, Pz, z);
            const int f = __shfl_sync(0xffffffffu, cntk, z);
            double best = -INFINITY;
#pragma unroll
            for (int j2 = 0; j2 < (LEAF ? NA : 1); ++j2) best = fmax(best, warp_sum_xor(Oz * Sv[j2]) / Pzz);
            const double Vz = a.qbar + best;
            accq += ((double)f / (double)a.n) * Vz;
            if (a.leafV && lane == 0) a.leafV[q * 16 + z] = Vz;
        }
        if (lane == 0) a.Q[q] = Rq + a.gamma * accq;
    }
}

// ---- child offsets: single-CTA exclusive scan -------------------------------------------------
__global__ void __launch_bounds__(1024) k_scan(const int32_t *__restrict__ U, int32_t *__restrict__ off, long long n,
                                               long long *total) {
    __shared__ long long wsum[32];
    __shared__ long long carry_s;
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

// ---- S4: Bayes correction of every unique z of a Q-node ----------------------------------------
struct CorrectArgs {
    const float *beliefs;
    long long bstride;
    const int32_t *vmap;
    const uint8_t *m8, *cell;
    const float *ctab, *O32;
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
    int H, W, HW, NAP, ntiles;
    float p_int, p_lat;
    long long qsel;   // >= 0: only this Q-node (belief_update)
};

template <uint32_t MASK>
__global__ void __launch_bounds__(256) k_correct(CorrectArgs a) {
    constexpr int NA = mask_count(MASK);
    const long long q = a.qsel >= 0 ? a.qsel : (long long)(blockIdx.x / a.ntiles);
    const int tile = blockIdx.x % a.ntiles;
    const long long w = q / NA;
    const int j = (int)(q % NA);
    const int k = action_of<MASK>(j);
    const long long v = a.vmap ? (long long)a.vmap[w] : w;
    const unsigned um = a.umask[q];
    const int U = __popc(um);
    const long long base = a.qsel >= 0 ? 0 : a.off[q];
    __shared__ float s_inv[16];
    __shared__ int s_z[16];
    if (threadIdx.x < 16) {
        const int z = threadIdx.x;
        if ((um >> z) & 1u) {
            const int rank = __popc(um & ((1u << z) - 1u));
            s_z[rank] = z;
            s_inv[rank] = (float)(1.0 / a.P[q * 16 + z]);
            if (tile == 0 && a.cpath) {
                const long long c = base + rank;
                a.cpath[c] = a.vpath[v] | ((uint64_t)(k + 1) << (8 * a.level)) | ((uint64_t)z << (8 * a.level + 4));
                a.cparent[c] = (int32_t)q;
                a.cz[c] = z;
                a.cf[c] = a.cnt[q * 16 + z];
                a.croot[c] = a.vroot[v];
            }
        }
    }
    __syncthreads();
    const long long x0 = ((long long)tile * blockDim.x + threadIdx.x) * 4;
    if (x0 >= a.HW) return;
    const float *__restrict__ b = a.beliefs + v * a.bstride;
    float bb[4];
    int sg[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const long long x = x0 + i;
        bb[i] = 0.f;
        sg[i] = 0;
        if (x >= a.HW) continue;
        const int ci = a.cell[x];
        sg[i] = ci & 15;
        if (ci & 16) continue;                      // occupied: bbar = 0
        const float b0 = b[x];
        if (k == 4) { bb[i] = b0; continue; }
        const int r = (int)(x / a.W), c = (int)(x % a.W);
        auto src = [&](int kk) -> float {           // b(y - d_kk), zero off-map
            const int rr = r - st_dr(kk), cc = c - st_dc(kk);
            if (rr < 0 || rr >= a.H || cc < 0 || cc >= a.W) return 0.f;
            return b[(long long)rr * a.W + cc];
        };
        const int m8 = a.m8[x];
        // runtime stencil id k: the laterals come from the ring (reading R3)
        const float s_int = src(k);
        const float s_lat = src(lat1(k)) + src(lat2(k));
        const float tt = a.ctab[m8 * a.NAP + j] * b0;
        bb[i] = fmaf(a.p_lat, s_lat, fmaf(a.p_int, s_int, tt));
    }
    const bool vec = ((a.cstride & 3) == 0) && (x0 + 3 < a.HW) && ((reinterpret_cast<uintptr_t>(a.child) & 15) == 0);
    for (int u = 0; u < U; ++u) {
        const int z = s_z[u];
        const float inv = s_inv[u];
        float o[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) o[i] = a.O32[sg[i] * 16 + z] * bb[i] * inv;
        float *dst = a.child + (base + u) * a.cstride + x0;
        if (vec) {
            *reinterpret_cast<float4 *>(dst) = make_float4(o[0], o[1], o[2], o[3]);
        } else {
#pragma unroll
            for (int i = 0; i < 4; ++i)
                if (x0 + i < a.HW) dst[i] = o[i];
        }
    }
}

// ---- S6 backup ---------------------------------------------------------------------------------
template <int NA>
__global__ void k_vmax(const double *__restrict__ Q, double *__restrict__ V, long long nwork, const int32_t *vmap) {
    const long long w = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (w >= nwork) return;
    double best = Q[w * NA];
#pragma unroll
    for (int j = 1; j < NA; ++j) best = fmax(best, Q[w * NA + j]);
    V[vmap ? vmap[w] : w] = best + 0.0;   // +0.0 canonicalises -0 for the exact zero-padded sum
}

template <int NA>
__global__ void k_backup(long long nwork, const int32_t *vmap, const double *__restrict__ R,
                         const uint16_t *__restrict__ umask, const int32_t *__restrict__ off,
                         const double *__restrict__ Vc, const int32_t *__restrict__ fc, int n, double gamma,
                         double *__restrict__ Q, double *__restrict__ V) {
    const long long w = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (w >= nwork) return;
    double best = -INFINITY;
#pragma unroll
    for (int j = 0; j < NA; ++j) {
        const long long q = w * NA + j;
        const int U = __popc((unsigned)umask[q]);
        const long long c0 = off[q];
        double acc = 0.0;
        for (int u = 0; u < U; ++u) acc += ((double)fc[c0 + u] / (double)n) * Vc[c0 + u];
        const double qv = R[q] + gamma * acc;   // Alg. 6 with gamma (R13)
        Q[q] = qv;
        best = fmax(best, qv);                  // Alg. 7
    }
    V[vmap ? vmap[w] : w] = best + 0.0;
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

// bracket one launch with instrumentation events (no-op unless profiling is on)
#define QVTS_PROF(cat, ...)                       \
    do {                                          \
        cudaEvent_t e__;                          \
        prof_begin(m, cat, st, &e__);             \
        __VA_ARGS__;                              \
        prof_end(m, cat, st, e__);                \
    } while (0)

template <uint32_t MASK, bool LEAF>
static size_t hist_smem(const BandSet &bs) {
    constexpr int NA = mask_count(MASK), NAP = (NA + 3) & ~3;
    const size_t region = std::max<size_t>(bs.tile_floats, (size_t)hist_nv<MASK, LEAF>() * (kHistThreads + 1));
    return (region + 256 * NAP) * sizeof(float);
}

template <uint32_t MASK, bool LEAF>
static qvts_status launch_hist(Model &m, const BandSet &bs, const float *beliefs, long long bstride,
                               const int32_t *vmap, long long nwork, int pstride, cudaStream_t st) {
    constexpr int NAP = (mask_count(MASK) + 3) & ~3;
    HistArgs a;
    a.beliefs = beliefs; a.bstride = bstride; a.vmap = vmap;
    a.bands = bs.bands.as<BandInfo>(); a.nb = bs.nb;
    a.entries = bs.entries.as<uint32_t>();
    a.qlist = bs.qlist.as<float4>();
    a.ctab = m.d_ctab.as<float>();
    a.H = m.H; a.W = m.W; a.TW = m.W + 2;
    a.region_floats = (int)std::max<size_t>(bs.tile_floats, (size_t)hist_nv<MASK, LEAF>() * (kHistThreads + 1));
    a.region_floats = (a.region_floats + 3) & ~3;
    a.p_int = (float)m.p_int; a.p_lat = (float)m.p_lat;
    a.part = m.part.as<double>(); a.pstride = pstride;
    const size_t smem = (a.region_floats + 256 * NAP) * sizeof(float);
    QVTS_CUDA(cudaFuncSetAttribute(k_hist<MASK, LEAF>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    const long long nblocks = nwork * bs.nb;
    if (nblocks > 0x7FFFFFFFLL) { set_error("too many hist blocks"); return QVTS_ERR_INVALID_ARG; }
    QVTS_PROF(LEAF ? 0 : 1, k_hist<MASK, LEAF><<<(unsigned)nblocks, kHistThreads, smem, st>>>(a));
    QVTS_CUDA(cudaGetLastError());
    (LEAF ? m.pstat.leaf_cells : m.pstat.hist_cells) += nwork * m.n_free;
    return QVTS_OK;
}

template <uint32_t MASK>
static int pstride_of(bool leaf) {
    constexpr int NA = mask_count(MASK);
    return 16 * NA * (leaf ? 1 + NA : 1) + NA + 1;
}

template <uint32_t MASK>
static qvts_status plan_levels_t(Model &m, const RootBatch &roots, const qvts_plan_cfg &cfg, const qvts_comm *comm,
                                 cudaStream_t st, long long *nv_out) {
    constexpr int NA = mask_count(MASK);
    const int D = cfg.depth, n = cfg.n_samples;
    const bool trace = cfg.want_trace != 0;
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

    for (int d = 0; d < D; ++d) {
        const bool leaf = (d == D - 1);
        VLevel &vl = m.vl[d];
        QLevel &ql = m.ql[d];
        const float *bel = d == 0 ? roots.beliefs : vl.belief.as<float>();
        const long long bstride = d == 0 ? roots.stride : m.HWp;
        // sharding: first level d >= 1 with >= shard_min V-nodes
        ql.mapped = false;
        long long nwork = vl.n;
        if (G > 1 && shard_level < 0 && d >= 1 && vl.n >= shard_min) {
            shard_level = d;
            nwork = vl.n > rank ? (vl.n - rank + G - 1) / G : 0;
            QVTS_TRY(ql.vmap.ensure(sizeof(int32_t) * std::max(1LL, nwork)));
            if (nwork) QVTS_PROF(7, k_iota_stride<<<nblk(nwork, 256), 256, 0, st>>>(ql.vmap.as<int32_t>(), nwork, rank, G));
            ql.mapped = true;
        }
        ql.nwork = nwork;
        const int32_t *vmap = ql.mapped ? ql.vmap.as<int32_t>() : nullptr;
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
            const BandSet &bs = (nwork * m.band_big.nb < 4 * 148) ? m.band_small : m.band_big;
            const int pstride = pstride_of<MASK>(leaf);
            QVTS_TRY(m.part.ensure(sizeof(double) * (size_t)nwork * bs.nb * pstride));
            if (leaf) QVTS_TRY((launch_hist<MASK, true>(m, bs, bel, bstride, vmap, nwork, pstride, st)));
            else QVTS_TRY((launch_hist<MASK, false>(m, bs, bel, bstride, vmap, nwork, pstride, st)));
            ReduceArgs r;
            r.part = m.part.as<double>(); r.pstride = pstride; r.nb = bs.nb; r.nq = nq; r.vmap = vmap;
            r.beliefs = bel; r.bstride = bstride; r.vpath = vl.path.as<uint64_t>(); r.vroot = vl.root.as<int32_t>();
            r.root_step = roots.step_dev; r.root_ep = roots.episode_dev; r.seed = cfg.seed;
            r.level = d; r.n = n; r.O64 = m.d_O64.as<double>();
            r.ngc = m.ngc; r.gc_cell = m.d_gc_cell.as<int32_t>(); r.gc_act = m.d_gc_act.as<int32_t>();
            r.gc_val = m.d_gc_val.as<double>(); r.goal = m.goal;
            r.p_stay = m.p_stay; r.gamma = m.gamma; r.qbar = m.qbar;
            r.R = ql.R.as<double>(); r.P = ql.P.as<double>(); r.cnt = ql.cnt.as<uint16_t>();
            r.umask = ql.umask.as<uint16_t>(); r.U = ql.U.as<int32_t>();
            r.zdraw = trace ? ql.zdraw.as<uint8_t>() : nullptr;
            r.Q = ql.Q.as<double>(); r.leafV = (trace && leaf) ? ql.leafV.as<double>() : nullptr;
            r.nflag = m.counters.as<unsigned long long>();
            if (leaf) QVTS_PROF(2, k_reduce<MASK, true><<<nblk(nq * 32, 256), 256, 0, st>>>(r));
            else QVTS_PROF(3, k_reduce<MASK, false><<<nblk(nq * 32, 256), 256, 0, st>>>(r));
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
            c.m8 = m.d_m8.as<uint8_t>(); c.cell = m.d_cell.as<uint8_t>(); c.ctab = m.d_ctab.as<float>();
            c.O32 = m.d_O32.as<float>(); c.P = ql.P.as<double>(); c.cnt = ql.cnt.as<uint16_t>();
            c.umask = ql.umask.as<uint16_t>(); c.off = ql.off.as<int32_t>();
            c.vpath = vl.path.as<uint64_t>(); c.vroot = vl.root.as<int32_t>(); c.level = d;
            c.child = vc.belief.as<float>(); c.cstride = m.HWp;
            c.cpath = vc.path.as<uint64_t>(); c.cparent = vc.parent_q.as<int32_t>(); c.cz = vc.z.as<int32_t>();
            c.cf = vc.f.as<int32_t>(); c.croot = vc.root.as<int32_t>();
            c.H = m.H; c.W = m.W; c.HW = m.HW; c.NAP = m.NAP;
            c.ntiles = (int)((m.HW + 1023) / 1024);
            c.p_int = (float)m.p_int; c.p_lat = (float)m.p_lat; c.qsel = -1;
            const long long nblocks = nq * c.ntiles;
            if (nblocks > 0x7FFFFFFFLL) { set_error("too many correct blocks"); return QVTS_ERR_INVALID_ARG; }
            QVTS_PROF(5, k_correct<MASK><<<(unsigned)nblocks, 256, 0, st>>>(c));
            QVTS_CUDA(cudaGetLastError());
            m.pstat.correct_cells_written += total * (long long)m.HW;
        }
    }
    // leaf V-node count (not materialised): sum of unique counts of the last Q-level
    {
        QLevel &ql = m.ql[D - 1];
        long long nq = ql.nwork * NA, total = 0;
        if (nq > 0) {
            QVTS_PROF(4, k_scan<<<1, 1024, 0, st>>>(ql.U.as<int32_t>(), ql.off.as<int32_t>(), nq, m.total.as<long long>()));
            QVTS_CUDA(cudaGetLastError());
            QVTS_CUDA(cudaMemcpyAsync(&total, m.total.p, sizeof(long long), cudaMemcpyDeviceToHost, st));
            QVTS_CUDA(cudaStreamSynchronize(st));
        }
        nv_out[D] = total;
    }
    // S6 backup, bottom-up
    for (int d = D - 1; d >= 0; --d) {
        QLevel &ql = m.ql[d];
        VLevel &vl = m.vl[d];
        const int32_t *vmap = ql.mapped ? ql.vmap.as<int32_t>() : nullptr;
        if (d == shard_level) QVTS_CUDA(cudaMemsetAsync(vl.V.p, 0, sizeof(double) * std::max(1LL, vl.n), st));
        if (ql.nwork > 0) {
            if (d == D - 1) {
                QVTS_PROF(6, k_vmax<NA><<<nblk(ql.nwork, 256), 256, 0, st>>>(ql.Q.as<double>(), vl.V.as<double>(), ql.nwork, vmap));
            } else {
                VLevel &vc = m.vl[d + 1];
                QVTS_PROF(6, k_backup<NA><<<nblk(ql.nwork, 256), 256, 0, st>>>(ql.nwork, vmap, ql.R.as<double>(),
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
    m.last_depth = D;
    m.last_shard_level = shard_level;
    m.last_n = n;
    m.last_trace = trace;
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
    if (!m || !root_dev || !cfg || !res) { set_error("NULL argument"); return QVTS_ERR_INVALID_ARG; }
    if (cfg->depth < 1 || cfg->depth > 8 || cfg->n_samples < 1 || cfg->n_samples > 4096) {
        set_error("depth must be 1..8 and n_samples 1..4096"); return QVTS_ERR_INVALID_ARG;
    }
    if (comm && (comm->nranks < 1 || comm->rank < 0 || comm->rank >= comm->nranks ||
                 (comm->nranks > 1 && !comm->allreduce_sum_f64))) {
        set_error("bad comm"); return QVTS_ERR_INVALID_ARG;
    }
    if (!m->have_q) { set_error("run qvts_value_iteration before planning"); return QVTS_ERR_STATE; }
    QVTS_CUDA(cudaSetDevice(m->device));
    cudaStream_t st = (cudaStream_t)stream;
    QVTS_TRY(m->ep_root_step.ensure(sizeof(uint32_t) * 2));
    QVTS_TRY(m->ep_root_ep.ensure(sizeof(uint32_t) * 2));
    uint32_t keys[2] = {cfg->step, cfg->episode};
    QVTS_CUDA(cudaMemcpyAsync(m->ep_root_step.p, &keys[0], sizeof(uint32_t), cudaMemcpyHostToDevice, st));
    QVTS_CUDA(cudaMemcpyAsync(m->ep_root_ep.p, &keys[1], sizeof(uint32_t), cudaMemcpyHostToDevice, st));
    RootBatch rb{root_dev, (long long)m->HW, 1, m->ep_root_step.as<uint32_t>(), m->ep_root_ep.as<uint32_t>()};
    long long nv[kMaxLevels + 1] = {0};
    QVTS_CUDA(cudaEventRecord(m->ev0, st));
    QVTS_TRY(plan_levels(*m, rb, *cfg, comm, st, nv));
    QVTS_CUDA(cudaEventRecord(m->ev1, st));
    double q[9];
    QVTS_CUDA(cudaMemcpyAsync(q, m->ql[0].Q.p, sizeof(double) * m->NA, cudaMemcpyDeviceToHost, st));
    QVTS_CUDA(cudaStreamSynchronize(st));
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
    return QVTS_OK;
}

extern "C" qvts_status qvts_belief_update(qvts_model *m, const float *b_dev, int32_t action, int32_t z,
                                          float *out_dev, double *p_obs_out, void *stream) {
    if (!m || !b_dev || !out_dev) { set_error("NULL argument"); return QVTS_ERR_INVALID_ARG; }
    int j = -1;
    for (int i = 0; i < m->NA; ++i) if (m->action_id[i] == action) j = i;
    if (j < 0 || z < 0 || z > 15) { set_error("action not in the action set or z out of range"); return QVTS_ERR_INVALID_ARG; }
    QVTS_CUDA(cudaSetDevice(m->device));
    cudaStream_t st = (cudaStream_t)stream;
    const int NA = m->NA;
    QVTS_TRY(m->bu_R.ensure(sizeof(double) * NA));
    QVTS_TRY(m->bu_P.ensure(sizeof(double) * 16 * NA));
    QVTS_TRY(m->bu_cnt.ensure(sizeof(uint16_t) * 16 * NA));
    QVTS_TRY(m->bu_umask.ensure(sizeof(uint16_t) * NA));
    QVTS_TRY(m->bu_U.ensure(sizeof(int32_t) * NA));
    QVTS_TRY(m->bu_off.ensure(sizeof(int32_t) * NA));
    QVTS_TRY(m->bu_path.ensure(sizeof(uint64_t)));
    QVTS_TRY(m->bu_root.ensure(sizeof(int32_t)));
    QVTS_TRY(m->bu_key.ensure(sizeof(uint32_t) * 2));
    QVTS_CUDA(cudaMemsetAsync(m->bu_path.p, 0, sizeof(uint64_t), st));
    QVTS_CUDA(cudaMemsetAsync(m->bu_root.p, 0, sizeof(int32_t), st));
    QVTS_CUDA(cudaMemsetAsync(m->bu_key.p, 0, sizeof(uint32_t) * 2, st));
    const BandSet &bs = m->band_small;
    qvts_status s = QVTS_ERR_INVALID_ARG;
#define QVTS_BU_HIST(MASK)                                                                                    \
    {                                                                                                         \
        const int ps = pstride_of<MASK>(false);                                                               \
        s = m->part.ensure(sizeof(double) * (size_t)bs.nb * ps);                                              \
        if (s == QVTS_OK) s = launch_hist<MASK, false>(*m, bs, b_dev, m->HW, nullptr, 1, ps, st);             \
        if (s == QVTS_OK) {                                                                                   \
            ReduceArgs r;                                                                                     \
            std::memset(&r, 0, sizeof(r));                                                                    \
            r.part = m->part.as<double>(); r.pstride = ps; r.nb = bs.nb; r.nq = NA;                           \
            r.beliefs = b_dev; r.bstride = m->HW; r.vpath = m->bu_path.as<uint64_t>();                        \
            r.vroot = m->bu_root.as<int32_t>(); r.root_step = m->bu_key.as<uint32_t>();                       \
            r.root_ep = m->bu_key.as<uint32_t>() + 1; r.n = 1; r.O64 = m->d_O64.as<double>();                 \
            r.ngc = m->ngc; r.gc_cell = m->d_gc_cell.as<int32_t>(); r.gc_act = m->d_gc_act.as<int32_t>();     \
            r.gc_val = m->d_gc_val.as<double>(); r.goal = m->goal; r.p_stay = m->p_stay; r.gamma = m->gamma;  \
            r.R = m->bu_R.as<double>(); r.P = m->bu_P.as<double>(); r.cnt = m->bu_cnt.as<uint16_t>();         \
            r.umask = m->bu_umask.as<uint16_t>(); r.U = m->bu_U.as<int32_t>();                                \
            k_reduce<MASK, false><<<nblk((long long)NA * 32, 256), 256, 0, st>>>(r);                          \
        }                                                                                                     \
    }
    QVTS_DISPATCH_MASK(m->mask, QVTS_BU_HIST);
#undef QVTS_BU_HIST
    QVTS_TRY(s);
    QVTS_CUDA(cudaGetLastError());
    double P[16];
    QVTS_CUDA(cudaMemcpyAsync(P, m->bu_P.as<double>() + 16 * j, sizeof(P), cudaMemcpyDeviceToHost, st));
    QVTS_CUDA(cudaStreamSynchronize(st));
    if (p_obs_out) *p_obs_out = P[z];
    if (!(P[z] > 1e-30)) { set_error("zero-likelihood observation"); return QVTS_ERR_ZERO_LIKELIHOOD; }
    uint16_t um = (uint16_t)(1u << z);
    std::vector<uint16_t> ums(NA, 0);
    ums[j] = um;
    QVTS_CUDA(cudaMemcpyAsync(m->bu_umask.p, ums.data(), sizeof(uint16_t) * NA, cudaMemcpyHostToDevice, st));
    CorrectArgs c;
    std::memset(&c, 0, sizeof(c));
    c.beliefs = b_dev; c.bstride = m->HW; c.m8 = m->d_m8.as<uint8_t>(); c.cell = m->d_cell.as<uint8_t>();
    c.ctab = m->d_ctab.as<float>(); c.O32 = m->d_O32.as<float>(); c.P = m->bu_P.as<double>();
    c.cnt = m->bu_cnt.as<uint16_t>(); c.umask = m->bu_umask.as<uint16_t>(); c.off = m->bu_off.as<int32_t>();
    c.vpath = m->bu_path.as<uint64_t>(); c.vroot = m->bu_root.as<int32_t>();
    c.child = out_dev; c.cstride = m->HW; c.H = m->H; c.W = m->W; c.HW = m->HW; c.NAP = m->NAP;
    c.ntiles = (int)((m->HW + 1023) / 1024); c.p_int = (float)m->p_int; c.p_lat = (float)m->p_lat; c.qsel = j;
#define QVTS_BU_CORR(MASK) k_correct<MASK><<<c.ntiles, 256, 0, st>>>(c)
    QVTS_DISPATCH_MASK(m->mask, QVTS_BU_CORR);
#undef QVTS_BU_CORR
    QVTS_CUDA(cudaGetLastError());
    QVTS_CUDA(cudaStreamSynchronize(st));
    return QVTS_OK;
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
        if (ql.mapped) { vmap.resize(ql.nwork); QVTS_TRY(d2h(vmap.data(), ql.vmap, vmap.size())); }
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
