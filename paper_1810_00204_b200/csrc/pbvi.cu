// pbvi.cu — PBVI lower bound (§IV-B), fp64, offline.
//
// Belief set: B0 = {b0}; each expansion round, every point b (in order) draws one Alg. 4 sample per
// action (x ~ b, x' ~ T(x,a,.), z ~ O(x',.) on Philox words 1..3 of counter (a, point, round,
// 0x7BB1), key (seed, 0xB5E7)); of the |A| posteriors Phi(b,a,z) the one farthest in L1 from the
// set as grown so far is added if that distance is > 0 (ties: lowest action).
// Backups: Gamma0 = {R_min/(1-gamma)}; a sweep gives every point b the vector
//   alpha_b = R(.,a*) + gamma sum_z g^{alpha*_{a*,z}}_{a*,z},
//   g^alpha_{a,z}(x) = sum_x' O(x',z) T(x,a,x') alpha(x'),
//   alpha*_{a,z} = argmax_alpha b . g^alpha_{a,z} = argmax_alpha sum_s O[s][z] sum_{sig(x')=s} bbar_a(x') alpha(x'),
//   a* = argmax_a [b . R(.,a) + gamma sum_z max_alpha b . g],   ties to the lowest index.
// The b . g values are signature-binned like the leaf kernel: Sc[b][a][s][k] over the free cells
// of class s (a static class-sorted cell list, split into chunks for a split-K fp64 product),
// then 16x16 O weights.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <vector>

#include "philox.cuh"
#include "qvts_internal.cuh"
#include "stencil.cuh"

namespace qvts {

// arg-max rule of reading B4: replace the incumbent only when larger by > 1e-10 (1 + |incumbent|)
__host__ __device__ __forceinline__ bool pb_beats(double v, double best) {
    return v > best + 1e-10 * (1.0 + fabs(best));
}

struct PbviDev {
    int HW, W, NA, P;                 // P = max points (alpha stride)
    double p_int, p_stay, p_lat, gamma, acc;
    const uint8_t *m8, *cell, *sig;   // cell = sig | occ << 4
    const double *O64, *R64;          // [16][16], [NA][HW]
};

// bbar_a(x) in fp64 (gather form of the clamped stencil, zero on occupied cells)
template <uint32_t MASK>
__device__ __forceinline__ double pb_predict(const PbviDev &d, const double *__restrict__ b, int x, int k) {
    if (d.cell[x] & 16) return 0.0;
    const double b0 = b[x];
    if (k == 4) return b0;
    const int m8 = d.m8[x];
    const int r = x / d.W, c = x % d.W, H = d.HW / d.W;
    auto h = [&](int kk) -> double {
        const int rr = r - st_dr(kk), cc = c - st_dc(kk);
        const double src = (rr >= 0 && rr < H && cc >= 0 && cc < d.W) ? b[rr * d.W + cc] : 0.0;
        return ((m8 >> nbit(kk)) & 1) ? src + b0 : src;
    };
    return d.p_stay * b0 + d.p_int * h(k) + d.p_lat * (h(lat1(k)) + h(lat2(k)));
}

template <uint32_t MASK>
__global__ void k_pb_predict(PbviDev d, const double *__restrict__ B, int nb, double *__restrict__ Bbar) {
    constexpr int NA = mask_count(MASK);
    const long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (t >= (long long)nb * d.HW) return;
    const int i = (int)(t / d.HW), x = (int)(t % d.HW);
    const double *b = B + (size_t)i * d.HW;
#pragma unroll
    for (int j = 0; j < NA; ++j) Bbar[((size_t)i * NA + j) * d.HW + x] = pb_predict<MASK>(d, b, x, mask_action(MASK, j));
}

// b . R(.,a) for every (point, action): one block each, fixed-order tree reduction
__global__ void k_pb_rb(PbviDev d, const double *__restrict__ B, double *__restrict__ Rb) {
    const int i = blockIdx.x / d.NA, j = blockIdx.x % d.NA;
    __shared__ double red[256];
    double s = 0.0;
    for (int x = threadIdx.x; x < d.HW; x += 256) s += d.R64[(size_t)j * d.HW + x] * B[(size_t)i * d.HW + x];
    red[threadIdx.x] = s;
    __syncthreads();
    for (int o = 128; o > 0; o >>= 1) {
        if (threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
        __syncthreads();
    }
    if (threadIdx.x == 0) Rb[blockIdx.x] = red[0];
}

// Sc as a split-K product over the class-sorted free cells: CTA (chunk, row block, vector block)
// takes one chunk (<= 64 cells of ONE class) and a 32 x 32 tile of (point-action row, alpha k),
// stages the gathered rows of bbar and the alpha columns in shared memory, and writes one fp64
// partial per (chunk, row, k); k_pb_bins_sum adds a class's chunks in order.
constexpr int kPbCh = 64;
__global__ void __launch_bounds__(256) k_pb_bins_part(const double *__restrict__ Bbar, int HW, int nrows,
                                                      const double *__restrict__ GT, int P, int nal,
                                                      const int32_t *__restrict__ cells,
                                                      const int2 *__restrict__ chunks, double *__restrict__ part,
                                                      int rows_pad) {
    __shared__ double Bs[32][kPbCh + 1];
    __shared__ double Gs[kPbCh][33];
    const int2 ch = chunks[blockIdx.x];                 // [e0, e1)
    const int n = ch.y - ch.x;
    const int r0 = blockIdx.y * 32, k0 = blockIdx.z * 32;
    const int t = threadIdx.x;
    for (int i = t; i < 32 * n; i += 256) {
        const int r = i / n, e = i % n;
        const int x = cells[ch.x + e];
        Bs[r][e] = (r0 + r < nrows) ? Bbar[(size_t)(r0 + r) * HW + x] : 0.0;
    }
    for (int i = t; i < n * 32; i += 256) {
        const int e = i >> 5, k = i & 31;
        const int x = cells[ch.x + e];
        Gs[e][k] = (k0 + k < nal) ? GT[(size_t)x * P + k0 + k] : 0.0;
    }
    __syncthreads();
    const int tr = t >> 4, tk = t & 15;                 // rows tr, tr+16; vectors tk, tk+16
    double a00 = 0.0, a01 = 0.0, a10 = 0.0, a11 = 0.0;
    for (int e = 0; e < n; ++e) {
        const double b0 = Bs[tr][e], b1 = Bs[tr + 16][e], g0 = Gs[e][tk], g1 = Gs[e][tk + 16];
        a00 = fma(b0, g0, a00); a01 = fma(b0, g1, a01);
        a10 = fma(b1, g0, a10); a11 = fma(b1, g1, a11);
    }
    double *out = part + (size_t)blockIdx.x * rows_pad * 32 * gridDim.z;
    const size_t pitch = (size_t)32 * gridDim.z;        // [chunk][row][k]
    out[(size_t)(r0 + tr) * pitch + k0 + tk] = a00;
    out[(size_t)(r0 + tr) * pitch + k0 + tk + 16] = a01;
    out[(size_t)(r0 + tr + 16) * pitch + k0 + tk] = a10;
    out[(size_t)(r0 + tr + 16) * pitch + k0 + tk + 16] = a11;
}

// Sc[row][s][k] = sum of class s's chunk partials in chunk order (zero for an empty class)
__global__ void k_pb_bins_sum(const double *__restrict__ part, const int32_t *__restrict__ cls_chunk, int nrows,
                              int nal, int P, int rows_pad, int kpad, double *__restrict__ Sc) {
    const long long tt = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (tt >= (long long)nrows * 16 * nal) return;
    const int k = (int)(tt % nal), s = (int)((tt / nal) % 16), r = (int)(tt / ((long long)nal * 16));
    double acc = 0.0;
    for (int c = cls_chunk[s]; c < cls_chunk[s + 1]; ++c) acc += part[((size_t)c * rows_pad + r) * kpad + k];
    Sc[((size_t)r * 16 + s) * P + k] = acc;
}

// per point: alpha*_{a,z} (lane z of warp a) and a* (ties: lowest index, strict >)
__global__ void k_pb_select(PbviDev d, const double *__restrict__ Sc, const double *__restrict__ Rb, int nal,
                            int32_t *__restrict__ sel, int32_t *__restrict__ astar) {
    const int i = blockIdx.x;
    const int lane = threadIdx.x & 31, a = threadIdx.x >> 5;
    __shared__ double va[9];
    if (a < d.NA) {
        double bz = 0.0;
        int bk = 0;
        if (lane < 16) {
            const double *S = Sc + ((size_t)i * d.NA + a) * 16 * d.P;
            for (int k = 0; k < nal; ++k) {
                double v = 0.0;
                for (int s = 0; s < 16; ++s) v += d.O64[s * 16 + lane] * S[(size_t)s * d.P + k];
                if (k == 0 || pb_beats(v, bz)) { bz = v; bk = k; }
            }
            sel[((size_t)i * d.NA + a) * 16 + lane] = bk;
        }
        double acc = 0.0;
        for (int z = 0; z < 16; ++z) acc += __shfl_sync(0xffffffffu, bz, z);
        if (lane == 0) va[a] = Rb[(size_t)i * d.NA + a] + d.gamma * acc;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        int best = 0;
        for (int j = 1; j < d.NA; ++j) if (pb_beats(va[j], va[best])) best = j;
        astar[i] = best;
    }
}

// alpha_i(x) = R(x,a*) + gamma sum_z sum_taps p_t O[sig(y_t)][z] alpha_{sel(z)}(y_t)
template <uint32_t MASK>
__global__ void k_pb_newalpha(PbviDev d, const double *__restrict__ G, int nb, const int32_t *__restrict__ sel,
                              const int32_t *__restrict__ astar, double *__restrict__ Gn) {
    constexpr int NA = mask_count(MASK);
    const long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (t >= (long long)nb * d.HW) return;
    const int i = (int)(t / d.HW), x = (int)(t % d.HW);
    const int j = astar[i];
    double out = 0.0;
    if (!(d.cell[x] & 16)) {
        int k = 0;
#pragma unroll
        for (int jj = 0; jj < NA; ++jj) if (jj == j) k = mask_action(MASK, jj);
        int ty[4];
        double tp[4];
        int nt;
        const int m8 = d.m8[x];
        auto tgt = [&](int kd) -> int {
            if ((m8 >> nbit(kd)) & 1) return x;
            return x + st_dr(kd) * d.W + st_dc(kd);
        };
        if (k == 4) { ty[0] = x; tp[0] = 1.0; nt = 1; }
        else {
            ty[0] = tgt(k); tp[0] = d.p_int;
            ty[1] = x; tp[1] = d.p_stay;
            ty[2] = tgt(lat1(k)); tp[2] = d.p_lat;
            ty[3] = tgt(lat2(k)); tp[3] = d.p_lat;
            nt = 4;
        }
        double acc = 0.0;
        for (int z = 0; z < 16; ++z) {
            const double *al = G + (size_t)sel[((size_t)i * NA + j) * 16 + z] * d.HW;
            double g = 0.0;
            for (int e = 0; e < nt; ++e) g += d.O64[d.sig[ty[e]] * 16 + z] * tp[e] * al[ty[e]];
            acc += g;
        }
        out = d.R64[(size_t)j * d.HW + x] + d.gamma * acc;
    }
    Gn[(size_t)i * d.HW + x] = out;
}

__global__ void k_pb_transpose(const double *__restrict__ G, int nal, int HW, int P, double *__restrict__ GT) {
    const long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (t >= (long long)nal * HW) return;
    const int k = (int)(t / HW), x = (int)(t % HW);
    GT[(size_t)x * P + k] = G[t];
}

__global__ void k_pb_fill(double *G, const uint8_t *__restrict__ cell, int HW, double v) {
    const int x = blockIdx.x * blockDim.x + threadIdx.x;
    if (x < HW) G[x] = (cell[x] & 16) ? 0.0 : v;
}

// ---- belief-set expansion pieces ----------------------------------------------------------------
// Alg. 4 on point b for every action: x ~ b (fp64 prefix over 256-cell chunks, word 1), x' ~ T
// (clamped row in stencil order, blocked targets merged into the stay entry; word 2), z ~ O (word 3).
template <uint32_t MASK>
__global__ void __launch_bounds__(256) k_pb_draw(PbviDev d, const double *__restrict__ b, int point, int round,
                                                 uint32_t seed, int32_t *__restrict__ zout) {
    constexpr int NA = mask_count(MASK);
    extern __shared__ double sx[];
    const int nch = (d.HW + 255) / 256;
    double *csum = sx, *cpre = sx + nch;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int c = warp; c < nch; c += 8) {
        double s = 0.0;
        for (int i = lane; i < 256; i += 32) {
            const int x = c * 256 + i;
            if (x < d.HW) s += b[x];
        }
        for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        if (lane == 0) csum[c] = s;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double acc = 0.0;
        for (int c = 0; c < nch; ++c) { cpre[c] = acc; acc += csum[c]; }
        cpre[nch] = acc;
    }
    __syncthreads();
    const int j = threadIdx.x;
    if (j >= NA) return;
    int k = 0;
#pragma unroll
    for (int jj = 0; jj < NA; ++jj) if (jj == j) k = mask_action(MASK, jj);
    const uint4 r = philox4x32_10(make_uint4((uint32_t)j, (uint32_t)point, (uint32_t)round, 0x7BB1u),
                                  make_uint2(seed, 0xB5E7u));
    const double t = philox_uniform(r.y) * cpre[nch];
    int lo = 0, hi = nch - 1;
    while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (t < cpre[mid + 1]) hi = mid; else lo = mid + 1;
    }
    double acc = cpre[lo];
    int x = -1, last = -1;
    for (int i = 0; i < 256; ++i) {
        const int xx = lo * 256 + i;
        if (xx >= d.HW) break;
        acc += b[xx];
        if (b[xx] > 0.0) last = xx;
        if (t < acc) { x = xx; break; }
    }
    if (x < 0) x = last >= 0 ? last : lo * 256;
    // x' ~ T(x,a,.) in the clamped row's stencil order
    int ty[4];
    double tp[4];
    int nt = 0;
    const int m8 = d.m8[x];
    for (int kk = 0; kk < 9; ++kk) {
        double wgt = 0.0;
        if (k == 4) wgt = (kk == 4) ? 1.0 : 0.0;
        else if (kk == k) wgt = d.p_int;
        else if (kk == 4) wgt = d.p_stay;
        else if (kk == lat1(k) || kk == lat2(k)) wgt = d.p_lat;
        if (wgt == 0.0) continue;
        int y = x;
        if (kk != 4 && !((m8 >> nbit(kk)) & 1)) y = x + st_dr(kk) * d.W + st_dc(kk);
        int found = -1;
        for (int e = 0; e < nt; ++e) if (ty[e] == y) found = e;
        if (found >= 0) tp[found] += wgt;
        else { ty[nt] = y; tp[nt] = wgt; ++nt; }
    }
    double C[4];
    acc = 0.0;
    for (int e = 0; e < nt; ++e) { acc += tp[e]; C[e] = acc; }
    double tt = philox_uniform(r.z) * C[nt - 1];
    int xp = ty[nt - 1];
    for (int e = 0; e < nt; ++e) if (tt < C[e]) { xp = ty[e]; break; }
    const int sg = d.sig[xp];
    double Cz[16];
    acc = 0.0;
    for (int z = 0; z < 16; ++z) {
        double o = 1.0;
        for (int bb = 0; bb < 4; ++bb) o *= (((z >> bb) & 1) == ((sg >> bb) & 1)) ? d.acc : (1.0 - d.acc);
        acc += o;
        Cz[z] = acc;
    }
    tt = philox_uniform(r.w) * Cz[15];
    int z = 15;
    for (int zz = 0; zz < 16; ++zz) if (tt < Cz[zz]) { z = zz; break; }
    zout[j] = z;
}

// candidate numerators O(x,z_a) bbar_a(x) and their sums P_a(z_a) (block per action, fixed order)
template <uint32_t MASK>
__global__ void k_pb_cand(PbviDev d, const double *__restrict__ b, const int32_t *__restrict__ zs,
                          double *__restrict__ cand, double *__restrict__ Pz) {
    constexpr int NA = mask_count(MASK);
    const int j = blockIdx.x;
    int k = 0;
#pragma unroll
    for (int jj = 0; jj < NA; ++jj) if (jj == j) k = mask_action(MASK, jj);
    const int z = zs[j];
    __shared__ double red[256];
    double s = 0.0;
    for (int x = threadIdx.x; x < d.HW; x += 256) {
        double v = 0.0;
        if (!(d.cell[x] & 16)) v = d.O64[(d.cell[x] & 15) * 16 + z] * pb_predict<MASK>(d, b, x, k);
        cand[(size_t)j * d.HW + x] = v;
        s += v;
    }
    red[threadIdx.x] = s;
    __syncthreads();
    for (int o = 128; o > 0; o >>= 1) {
        if (threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
        __syncthreads();
    }
    if (threadIdx.x == 0) Pz[j] = red[0];
}

__global__ void k_pb_normalise(double *cand, const double *__restrict__ Pz, int NA, int HW) {
    const long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (t >= (long long)NA * HW) return;
    const int j = (int)(t / HW);
    const double p = Pz[j];
    cand[t] = p > 1e-300 ? cand[t] / p : 0.0;
}

// L1 distance of every candidate to every point: block per (candidate, point), fixed order
__global__ void k_pb_l1(const double *__restrict__ cand, const double *__restrict__ B, int nb, int HW,
                        double *__restrict__ dist) {
    const int j = blockIdx.x / nb, k = blockIdx.x % nb;
    __shared__ double red[256];
    double s = 0.0;
    for (int x = threadIdx.x; x < HW; x += 256) s += fabs(cand[(size_t)j * HW + x] - B[(size_t)k * HW + x]);
    red[threadIdx.x] = s;
    __syncthreads();
    for (int o = 128; o > 0; o >>= 1) {
        if (threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
        __syncthreads();
    }
    if (threadIdx.x == 0) dist[blockIdx.x] = red[0];
}

template <uint32_t MASK>
static qvts_status pbvi_run(Model &m, const double *b0_dev, int expansions, int max_points, uint32_t seed,
                            int sweeps, cudaStream_t st) {
    constexpr int NA = mask_count(MASK);
    const int HW = m.HW;
    const int P = std::max(1, max_points);
    PbviDev d;
    d.HW = HW; d.W = m.W; d.NA = NA; d.P = P;
    d.p_int = m.p_int; d.p_stay = m.p_stay; d.p_lat = m.p_lat; d.gamma = m.gamma; d.acc = m.acc;
    d.m8 = m.d_m8.as<uint8_t>(); d.cell = m.d_cell.as<uint8_t>(); d.sig = m.d_sig.as<uint8_t>();
    d.O64 = m.d_O64.as<double>(); d.R64 = m.d_R64.as<double>();
    QVTS_TRY(m.pb_B.ensure(sizeof(double) * (size_t)P * HW));
    QVTS_TRY(m.pb_G.ensure(sizeof(double) * (size_t)P * HW));
    QVTS_TRY(m.pb_Gn.ensure(sizeof(double) * (size_t)P * HW));
    QVTS_TRY(m.pb_GT.ensure(sizeof(double) * (size_t)P * HW));
    QVTS_TRY(m.pb_Bbar.ensure(sizeof(double) * (size_t)P * NA * HW));
    QVTS_TRY(m.pb_Sc.ensure(sizeof(double) * (size_t)P * NA * 16 * P));
    QVTS_TRY(m.pb_Rb.ensure(sizeof(double) * (size_t)P * NA));
    QVTS_TRY(m.pb_sel.ensure(sizeof(int32_t) * (size_t)P * NA * 16));
    QVTS_TRY(m.pb_astar.ensure(sizeof(int32_t) * P));
    QVTS_TRY(m.pb_cand.ensure(sizeof(double) * (size_t)NA * HW));
    QVTS_TRY(m.pb_misc.ensure(sizeof(double) * (size_t)(NA + NA * P + NA)));
    // class-sorted free cells (static)
    std::vector<int32_t> cells, off(17, 0);
    for (int s = 0; s < 16; ++s) {
        off[s] = (int32_t)cells.size();
        for (int x = 0; x < HW; ++x) if (!m.occ[x] && m.sig[x] == s) cells.push_back(x);
    }
    off[16] = (int32_t)cells.size();
    // chunks of <= kPbCh cells that never cross a class boundary, and each class's chunk range
    std::vector<int2> chunks;
    std::vector<int32_t> cls_chunk(17, 0);
    for (int s2 = 0; s2 < 16; ++s2) {
        cls_chunk[s2] = (int32_t)chunks.size();
        for (int e0 = off[s2]; e0 < off[s2 + 1]; e0 += kPbCh) chunks.push_back(make_int2(e0, std::min(off[s2 + 1], e0 + kPbCh)));
    }
    cls_chunk[16] = (int32_t)chunks.size();
    QVTS_TRY(m.pb_chunks.ensure(sizeof(int2) * std::max<size_t>(1, chunks.size()) + sizeof(int32_t) * 17));
    QVTS_CUDA(cudaMemcpyAsync(m.pb_chunks.p, chunks.data(), sizeof(int2) * chunks.size(), cudaMemcpyHostToDevice, st));
    int32_t *d_cls_chunk = reinterpret_cast<int32_t *>(m.pb_chunks.as<int2>() + std::max<size_t>(1, chunks.size()));
    QVTS_CUDA(cudaMemcpyAsync(d_cls_chunk, cls_chunk.data(), sizeof(int32_t) * 17, cudaMemcpyHostToDevice, st));
    QVTS_TRY(m.pb_cls.ensure(sizeof(int32_t) * (cells.size() + 17)));
    QVTS_CUDA(cudaMemcpyAsync(m.pb_cls.p, off.data(), sizeof(int32_t) * 17, cudaMemcpyHostToDevice, st));
    QVTS_CUDA(cudaMemcpyAsync(m.pb_cls.as<int32_t>() + 17, cells.data(), sizeof(int32_t) * cells.size(),
                              cudaMemcpyHostToDevice, st));
    double *B = m.pb_B.as<double>();
    QVTS_CUDA(cudaMemcpyAsync(B, b0_dev, sizeof(double) * HW, cudaMemcpyDeviceToDevice, st));
    int nb = 1;
    // ---- belief-set expansion (sequential over points, as defined) ----
    double *cand = m.pb_cand.as<double>();
    double *Pz = m.pb_misc.as<double>(), *dist = Pz + NA;
    int32_t *zs = m.pb_sel.as<int32_t>();
    const int nch = (HW + 255) / 256;
    std::vector<double> hP(NA), hd;
    for (int r = 0; r < expansions && nb < P; ++r) {
        const int n0 = nb;
        for (int i = 0; i < n0 && nb < P; ++i) {
            const double *b = B + (size_t)i * HW;
            k_pb_draw<MASK><<<1, 256, sizeof(double) * (2 * nch + 1), st>>>(d, b, i, r, seed, zs);
            k_pb_cand<MASK><<<NA, 256, 0, st>>>(d, b, zs, cand, Pz);
            k_pb_normalise<<<(unsigned)(((long long)NA * HW + 255) / 256), 256, 0, st>>>(cand, Pz, NA, HW);
            k_pb_l1<<<NA * nb, 256, 0, st>>>(cand, B, nb, HW, dist);
            QVTS_CUDA(cudaGetLastError());
            hd.resize((size_t)NA * nb);
            QVTS_CUDA(cudaMemcpyAsync(hP.data(), Pz, sizeof(double) * NA, cudaMemcpyDeviceToHost, st));
            QVTS_CUDA(cudaMemcpyAsync(hd.data(), dist, sizeof(double) * NA * nb, cudaMemcpyDeviceToHost, st));
            QVTS_CUDA(cudaStreamSynchronize(st));
            int best_a = -1;
            double best_d = 0.0;
            for (int j = 0; j < NA; ++j) {
                if (!(hP[j] > 1e-300)) continue;            // zero-likelihood candidate: skipped
                double dmin = INFINITY;
                for (int k = 0; k < nb; ++k) dmin = std::min(dmin, hd[(size_t)j * nb + k]);
                if (pb_beats(dmin, best_d)) { best_d = dmin; best_a = j; }
            }
            if (best_a >= 0) {
                QVTS_CUDA(cudaMemcpyAsync(B + (size_t)nb * HW, cand + (size_t)best_a * HW, sizeof(double) * HW,
                                          cudaMemcpyDeviceToDevice, st));
                ++nb;
            }
        }
    }
    // ---- point-based backups from the blind lower bound ----
    double rmin = INFINITY;
    for (size_t i = 0; i < m.R64.size(); ++i)
        if (!m.occ[i % HW]) rmin = std::min(rmin, m.R64[i]);
    double *G = m.pb_G.as<double>(), *Gn = m.pb_Gn.as<double>(), *GT = m.pb_GT.as<double>();
    k_pb_fill<<<(HW + 255) / 256, 256, 0, st>>>(G, d.cell, HW, rmin / (1.0 - m.gamma));
    int nal = 1;
    std::vector<int32_t> ast(nb);
    std::vector<int32_t> gact(nb, 0);   // as the oracle before any sweep
    const long long nbx = (long long)nb * HW;
    k_pb_predict<MASK><<<(unsigned)((nbx + 255) / 256), 256, 0, st>>>(d, B, nb, m.pb_Bbar.as<double>());
    k_pb_rb<<<nb * NA, 256, 0, st>>>(d, B, m.pb_Rb.as<double>());
    for (int sw = 0; sw < sweeps; ++sw) {
        k_pb_transpose<<<(unsigned)(((long long)nal * HW + 255) / 256), 256, 0, st>>>(G, nal, HW, P, GT);
        {
            const int nrows = nb * NA, rows_pad = ((nrows + 31) / 32) * 32, kb = (nal + 31) / 32;
            const size_t nch = chunks.size();
            if (nch > 0) {
                QVTS_TRY(m.pb_part.ensure(sizeof(double) * nch * rows_pad * 32 * kb));
                k_pb_bins_part<<<dim3((unsigned)nch, rows_pad / 32, kb), 256, 0, st>>>(
                    m.pb_Bbar.as<double>(), HW, nrows, GT, P, nal, m.pb_cls.as<int32_t>() + 17, m.pb_chunks.as<int2>(),
                    m.pb_part.as<double>(), rows_pad);
            }
            const long long nout = (long long)nrows * 16 * nal;
            k_pb_bins_sum<<<(unsigned)((nout + 255) / 256), 256, 0, st>>>(m.pb_part.as<double>(), d_cls_chunk, nrows,
                                                                         nal, P, rows_pad, 32 * kb,
                                                                         m.pb_Sc.as<double>());
        }
        k_pb_select<<<nb, NA * 32, 0, st>>>(d, m.pb_Sc.as<double>(), m.pb_Rb.as<double>(), nal, m.pb_sel.as<int32_t>(),
                                            m.pb_astar.as<int32_t>());
        k_pb_newalpha<MASK><<<(unsigned)((nbx + 255) / 256), 256, 0, st>>>(d, G, nb, m.pb_sel.as<int32_t>(),
                                                                          m.pb_astar.as<int32_t>(), Gn);
        QVTS_CUDA(cudaGetLastError());
        std::swap(G, Gn);
        nal = nb;
    }
    if (sweeps > 0) {
        QVTS_CUDA(cudaMemcpyAsync(ast.data(), m.pb_astar.p, sizeof(int32_t) * nb, cudaMemcpyDeviceToHost, st));
        QVTS_CUDA(cudaStreamSynchronize(st));
        for (int i = 0; i < nb; ++i) gact[i] = m.action_id[ast[i]];
    }
    if (G != m.pb_G.as<double>())
        QVTS_CUDA(cudaMemcpyAsync(m.pb_G.p, G, sizeof(double) * (size_t)nal * HW, cudaMemcpyDeviceToDevice, st));
    // keep a transposed copy for bound evaluation
    k_pb_transpose<<<(unsigned)(((long long)nal * HW + 255) / 256), 256, 0, st>>>(m.pb_G.as<double>(), nal, HW, P, GT);
    QVTS_CUDA(cudaGetLastError());
    QVTS_CUDA(cudaStreamSynchronize(st));
    m.pb_np = nb;
    m.pb_nal = nal;
    m.pb_P = P;
    m.pb_act = gact;
    m.have_pbvi = true;
    return QVTS_OK;
}

}  // namespace qvts

using namespace qvts;

extern "C" qvts_status qvts_pbvi(qvts_model *m, const float *b0_dev, int32_t expansions, int32_t max_points,
                                 uint32_t seed, int32_t sweeps, int32_t *n_points_out, void *stream) {
    qvts::NvtxRange nvtx_range__("qvts_pbvi");
    if (!m || expansions < 0 || max_points < 1 || max_points > 1024 || sweeps < 0) {
        set_error("bad pbvi arguments");
        return QVTS_ERR_INVALID_ARG;
    }
    QVTS_CUDA(cudaSetDevice(m->device));
    cudaStream_t st = (cudaStream_t)stream;
    // b0 in fp64 (uniform over free cells when NULL)
    std::vector<double> hb(m->HW, 0.0);
    if (b0_dev) {
        std::vector<float> hf(m->HW);
        QVTS_CUDA(cudaMemcpy(hf.data(), b0_dev, sizeof(float) * m->HW, cudaMemcpyDeviceToHost));
        for (int x = 0; x < m->HW; ++x) hb[x] = hf[x];
    } else {
        for (int x = 0; x < m->HW; ++x) hb[x] = m->occ[x] ? 0.0 : 1.0 / (double)m->n_free;
    }
    QVTS_TRY(m->pb_b0.ensure(sizeof(double) * m->HW));
    QVTS_CUDA(cudaMemcpy(m->pb_b0.p, hb.data(), sizeof(double) * m->HW, cudaMemcpyHostToDevice));
    qvts_status s = QVTS_ERR_INVALID_ARG;
#define QVTS_PB(MASK) s = pbvi_run<MASK>(*m, m->pb_b0.as<double>(), expansions, max_points, seed, sweeps, st)
    QVTS_DISPATCH_MASK(m->mask, QVTS_PB);
#undef QVTS_PB
    if (s == QVTS_OK && n_points_out) *n_points_out = m->pb_np;
    return s;
}

extern "C" qvts_status qvts_get_pbvi(const qvts_model *m, double *points_host, double *alpha_host,
                                     int32_t *actions_host, int32_t *n_alpha_out) {
    if (!m) { set_error("model is NULL"); return QVTS_ERR_INVALID_ARG; }
    if (!m->have_pbvi) { set_error("qvts_pbvi has not run"); return QVTS_ERR_STATE; }
    QVTS_CUDA(cudaSetDevice(m->device));
    if (points_host)
        QVTS_CUDA(cudaMemcpy(points_host, m->pb_B.p, sizeof(double) * (size_t)m->pb_np * m->HW, cudaMemcpyDeviceToHost));
    if (alpha_host)
        QVTS_CUDA(cudaMemcpy(alpha_host, m->pb_G.p, sizeof(double) * (size_t)m->pb_nal * m->HW, cudaMemcpyDeviceToHost));
    if (actions_host) std::memcpy(actions_host, m->pb_act.data(), sizeof(int32_t) * m->pb_act.size());
    if (n_alpha_out) *n_alpha_out = m->pb_nal;
    return QVTS_OK;
}
