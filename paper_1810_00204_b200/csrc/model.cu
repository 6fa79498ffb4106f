// model.cu — qvts_model_create / destroy, compiled grid tables, class-partitioned band lists,
// and the fp64 value-iteration kernels (K1) behind qvts_value_iteration.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>

#include "qvts_internal.cuh"
#include "stencil.cuh"

namespace qvts {

static thread_local std::string g_last_error;
void set_error(const std::string &msg) { g_last_error = msg; }

qvts_status DevBuf::ensure(size_t bytes) {
    if (bytes <= cap && p) return QVTS_OK;
    release();
    // headroom: tree levels vary from step to step; regrowing (cudaFree + cudaMalloc of tens of
    // GB) would stall the device every time a step's tree is a little larger
    size_t want = std::max<size_t>(bytes + bytes / 4, 256);
    cudaError_t e = cudaMalloc(&p, want);
    if (e != cudaSuccess && want > bytes) {      // no room for headroom: exact size
        cudaGetLastError();
        want = std::max<size_t>(bytes, 256);
        e = cudaMalloc(&p, want);
    }
    if (e != cudaSuccess) {
        p = nullptr;
        cap = 0;
        cudaGetLastError();
        set_error("cudaMalloc(" + std::to_string(want) + " B): " + cudaGetErrorString(e));
        return e == cudaErrorMemoryAllocation ? QVTS_ERR_OUT_OF_MEMORY : QVTS_ERR_CUDA;
    }
    cap = want;
    return QVTS_OK;
}
void DevBuf::release() {
    if (p) cudaFree(p);
    p = nullptr;
    cap = 0;
}

qvts_status HostBuf::ensure(size_t bytes) {
    if (bytes <= cap && p) return QVTS_OK;
    release();
    const size_t want = std::max<size_t>(bytes + bytes / 4, 4096);
    if (cudaHostAlloc(&p, want, cudaHostAllocDefault) != cudaSuccess) {
        cudaGetLastError();
        p = nullptr;
        set_error("cudaHostAlloc failed");
        return QVTS_ERR_CUDA;
    }
    cap = want;
    return QVTS_OK;
}

void HostBuf::release() {
    if (p) cudaFreeHost(p);
    p = nullptr;
    cap = 0;
}


// ---- instrumentation -----------------------------------------------------------------------------
static cudaEvent_t next_event(Model &m) {
    if (m.evnext == m.evpool.size()) {
        cudaEvent_t e;
        if (cudaEventCreate(&e) != cudaSuccess) return nullptr;
        m.evpool.push_back(e);
    }
    return m.evpool[m.evnext++];
}
void prof_begin(Model &m, int cat, cudaStream_t st, cudaEvent_t *out) {
    (void)cat;
    *out = nullptr;
    m.pstat.total_launches++;
    if (!m.prof) return;
    *out = next_event(m);
    if (*out) cudaEventRecord(*out, st);
}
void prof_end(Model &m, int cat, cudaStream_t st, cudaEvent_t a) {
    if (!m.prof || !a) return;
    cudaEvent_t b = next_event(m);
    if (!b) return;
    cudaEventRecord(b, st);
    m.evrecs.push_back({cat, a, b});
}
void prof_collect(Model &m) {
    for (auto &r : m.evrecs) {
        float ms = 0.f;
        if (cudaEventElapsedTime(&ms, r.a, r.b) == cudaSuccess) {
            m.pstat.ms[r.cat] += ms;
            m.pstat.launches[r.cat]++;
        }
    }
    cudaGetLastError();
    m.evrecs.clear();
    m.evnext = 0;
}

// ---- class-partitioned band lists -----------------------------------------------------------
// For every band of `rows` grid rows, the free cells are grouped by wall signature sig (the
// observation class of Eq. 3's O(x', z)).  Class c receives k_c threads; thread j
// of class c takes the class-c cells j, j+k_c, ... in raster order, padded to L slots with
// entry 0 (tile cell 0 is a zero halo cell, so pads contribute exact zeros).
// Entry word: bits 0..15 tile index (halo-padded tile of width W+2), bits 16..23 the
// 8-neighbour occupancy byte m8.
qvts_status build_bands(Model &m, BandSet &bs, int rows) {
    const int T = kHistThreads;
    const int H = m.H, W = m.W, TW = (W + 5 + 3) & ~3;   // row pitch; grid column c at tile column c + 4
    rows = std::max(1, std::min(rows, H));
    // two parents' tiles per hist CTA must fit in shared memory (~190 KB) and index in 16 bits
    while (rows > 1 && ((long long)(rows + 5) * TW > 65535 || (long long)(rows + 5) * TW * 8 > 100000)) --rows;
    if ((long long)(rows + 2) * TW > 65535) {
        set_error("grid too wide for the band tile (W+2)*3 > 65535");
        return QVTS_ERR_INVALID_ARG;
    }
    bs.rows = rows;
    bs.nb = (H + rows - 1) / rows;
    bs.tile_floats = (rows + 2 + 3) * TW;      // + 3 zero rows holding the padding cell
    bs.tile_pitch = TW;
    bs.h_bands.assign(bs.nb, BandInfo{});
    std::vector<uint32_t> entries;
    bs.h_slot_cell.clear();
    long long off = 0;
    for (int b = 0; b < bs.nb; ++b) {
        BandInfo &bi = bs.h_bands[b];
        bi.row0 = b * rows;
        bi.nrows = std::min(rows, H - bi.row0);
        std::vector<int> cls[16];
        for (int r = bi.row0; r < bi.row0 + bi.nrows; ++r)
            for (int c = 0; c < W; ++c) {
                int x = r * W + c;
                if (!m.occ[x]) cls[m.sig[x]].push_back(x);
            }
        // smallest L with sum_c ceil(n_c / L) <= T
        int total = 0;
        for (int c = 0; c < 16; ++c) total += (int)cls[c].size();
        int L = std::max(1, (total + T - 1) / T);
        for (;; ++L) {
            int need = 0;
            for (int c = 0; c < 16; ++c) need += ((int)cls[c].size() + L - 1) / L;
            if (need <= T) break;
        }
        if (total == 0) L = 1;
        // L rounded to the kernel's 2-cell unroll, plus trailing pad steps for its look-ahead loads
        const int Lpad = ((L + 1) & ~1) + 4;
        bi.L = (L + 1) & ~1;
        bi.slot_off = off;
        // padding slots point at a cell of the 3 zero rows after the tile (zero neighbourhood)
        const uint32_t pad_e = (uint32_t)((bi.nrows + 2 + 1) * TW + 5);
        // thread ranges per class
        std::vector<int> cls_of(T, -1);
        int t0 = 0;
        for (int c = 0; c < 16; ++c) {
            bi.cs[c] = t0;
            const int k = ((int)cls[c].size() + L - 1) / L;
            for (int j = 0; j < k; ++j) cls_of[t0 + j] = c;
            t0 += k;
        }
        // Deal the cells step by step.  Within each group of 16 slot-threads (one half-warp per
        // parent) the 16 cells of a step get distinct tile residues mod 16, so the 9 neighbour
        // loads of a warp hit 32 distinct shared-memory banks (the second parent's tile sits 16
        // banks further).
        std::vector<std::vector<int>> bucket[16];
        std::vector<size_t> head[16];
        for (int c = 0; c < 16; ++c) {
            bucket[c].assign(16, {});
            head[c].assign(16, 0);
            for (int x : cls[c]) {
                int r = x / W, cc = x % W;
                int ti = (r - bi.row0 + 1) * TW + (cc + 4);
                bucket[c][ti & 15].push_back(x);
            }
        }
        std::vector<uint32_t> e((size_t)Lpad * T, pad_e);
        std::vector<int32_t> sc((size_t)Lpad * T, -1);
        for (int step = 0; step < L; ++step)
            for (int g = 0; g < T / 16; ++g) {
                unsigned used = 0;
                for (int tt = 16 * g; tt < 16 * g + 16; ++tt) {
                    const int c = cls_of[tt];
                    if (c < 0) continue;
                    int best = -1, bestn = 0, anyr = -1, anyn = 0;
                    for (int r = 0; r < 16; ++r) {
                        int left = (int)(bucket[c][r].size() - head[c][r]);
                        if (left <= 0) continue;
                        if (!(used >> r & 1) && left > bestn) { best = r; bestn = left; }
                        if (left > anyn) { anyr = r; anyn = left; }
                    }
                    if (best < 0) best = anyr;
                    if (best < 0) continue;            // class exhausted: padding slot
                    const int x = bucket[c][best][head[c][best]++];
                    used |= 1u << best;
                    int r = x / W, cc = x % W;
                    int ti = (r - bi.row0 + 1) * TW + (cc + 4);
                    e[(size_t)step * T + tt] = (uint32_t)ti | ((uint32_t)m.m8[x] << 16);
                    sc[(size_t)step * T + tt] = x;
                }
            }
        bi.cs[16] = t0;
        entries.insert(entries.end(), e.begin(), e.end());
        bs.h_slot_cell.insert(bs.h_slot_cell.end(), sc.begin(), sc.end());
        off += (long long)Lpad * T;
    }
    bs.total_slots = off;
    QVTS_TRY(upload(bs.bands, bs.h_bands));
    QVTS_TRY(upload(bs.entries, entries));
    QVTS_TRY(upload(bs.slot_cell, bs.h_slot_cell));
    return QVTS_OK;
}

// Q in slot order, offset by qbar (SURVEY c.6 rule 5): qlist[slot][NAP].
// T > 0: the leaf kernel's layout [step][NAP / 4][T slots][4] (slot s = step * T + t), so a warp's
// 16-byte copies of one quarter-row are contiguous
__global__ void k_qlist(const double *__restrict__ Q64, const int32_t *__restrict__ slot_cell,
                        long long nslots, int NA, int NAP, int HW, double qbar, float *__restrict__ out, int T = 0) {
    long long s = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (s >= nslots) return;
    int x = slot_cell[s];
    for (int j = 0; j < NAP; ++j) {
        float v = 0.f;
        if (x >= 0 && j < NA) v = (float)(Q64[(size_t)j * HW + x] - qbar);
        if (T > 0) out[(((s / T) * (NAP / 4) + j / 4) * T + s % T) * 4 + (j & 3)] = v;
        else out[s * NAP + j] = v;
    }
}

qvts_status build_qlists(Model &m, const double *src64, double qbar, bool fib, cudaStream_t st) {
    for (BandSet *bs : {&m.band_big, &m.band_small}) {
        DevBuf &dst = fib ? bs->qlist_fib : bs->qlist;
        QVTS_TRY(dst.ensure(sizeof(float) * bs->total_slots * m.NAP));
        long long n = bs->total_slots;
        k_qlist<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(src64, bs->slot_cell.as<int32_t>(), n, m.NA, m.NAP, m.HW,
                                                            qbar, dst.as<float>());
        QVTS_CUDA(cudaGetLastError());
    }
    {
        LeafBands &lb = m.leafb;
        DevBuf &dst = fib ? lb.qlist_fib : lb.qlist;
        QVTS_TRY(dst.ensure(sizeof(float) * lb.total_slots * m.NAP));
        const long long n = lb.total_slots;
        k_qlist<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(src64, lb.slot_cell.as<int32_t>(), n, m.NA, m.NAP, m.HW,
                                                            qbar, dst.as<float>(), kLeafThreads);
        QVTS_CUDA(cudaGetLastError());
    }
    return build_leaf_qfrag(m, src64, qbar, fib, st);
}

// ---- Fast Informed Bound (Eq. 7), fp64 -----------------------------------------
// One sweep, one thread per cell: for every action a, the clamped successor taps y_t with
// probabilities p_t (as in VI), then alpha'(x,a) = R(x,a) + gamma sum_z max_a' sum_t
// O[sig(y_t)][z] p_t alpha(y_t, a').  Occupied cells keep 0.  No-op once converged (as VI).
template <uint32_t MASK>
__global__ void __launch_bounds__(128) k_fib_sweep(const double *__restrict__ Ain, double *__restrict__ Aout,
                                                   const double *__restrict__ R64, const uint8_t *__restrict__ m8v,
                                                   const uint8_t *__restrict__ freev, const uint8_t *__restrict__ sigv,
                                                   const double *__restrict__ O64g, int HW, int W, double p_int,
                                                   double p_stay, double p_lat, double gamma,
                                                   unsigned long long *resid, int k, double eps) {
    if (k > 0 && __longlong_as_double((long long)resid[k - 1]) < eps) return;   // converged
    constexpr int NA = mask_count(MASK);
    __shared__ double sO[256];
    for (int i = threadIdx.x; i < 256; i += blockDim.x) sO[i] = O64g[i];
    __syncthreads();
    const int x = blockIdx.x * blockDim.x + threadIdx.x;
    double diff = 0.0;
    if (x < HW) {
        const bool fr = freev[x] != 0;
        const int m8 = m8v[x];
#pragma unroll 1
        for (int j = 0; j < NA; ++j) {
            double out = 0.0;
            if (fr) {
                int kk = 0;
#pragma unroll
                for (int i = 0; i < NA; ++i) if (i == j) kk = mask_action(MASK, i);
                int ty[4], ts[4];
                double tp[4];
                int nt;
                auto tgt = [&](int kd) -> int {
                    if ((m8 >> nbit(kd)) & 1) return x;
                    return x + st_dr(kd) * W + st_dc(kd);
                };
                if (kk == 4) {
                    ty[0] = x; tp[0] = 1.0; nt = 1;
                } else {
                    ty[0] = tgt(kk); tp[0] = p_int;
                    ty[1] = x; tp[1] = p_stay;
                    ty[2] = tgt(lat1(kk)); tp[2] = p_lat;
                    ty[3] = tgt(lat2(kk)); tp[3] = p_lat;
                    nt = 4;
                }
                double v[NA][4];
#pragma unroll
                for (int t = 0; t < 4; ++t) {
                    ts[t] = t < nt ? sigv[ty[t]] : 0;
#pragma unroll
                    for (int a2 = 0; a2 < NA; ++a2) v[a2][t] = t < nt ? tp[t] * Ain[(size_t)a2 * HW + ty[t]] : 0.0;
                }
                double s = 0.0;
                for (int z = 0; z < 16; ++z) {
                    const double o0 = sO[ts[0] * 16 + z], o1 = sO[ts[1] * 16 + z], o2 = sO[ts[2] * 16 + z],
                                 o3 = sO[ts[3] * 16 + z];
                    double best = -INFINITY;
#pragma unroll
                    for (int a2 = 0; a2 < NA; ++a2)
                        best = fmax(best, o0 * v[a2][0] + o1 * v[a2][1] + o2 * v[a2][2] + o3 * v[a2][3]);
                    s += best;
                }
                out = R64[(size_t)j * HW + x] + gamma * s;
            }
            Aout[(size_t)j * HW + x] = out;
            diff = fmax(diff, fabs(out - Ain[(size_t)j * HW + x]));
        }
    }
    for (int o = 16; o > 0; o >>= 1) diff = fmax(diff, __shfl_xor_sync(0xffffffffu, diff, o));
    if ((threadIdx.x & 31) == 0 && diff > 0.0)
        atomicMax(&resid[k], (unsigned long long)__double_as_longlong(diff));
}

__global__ void k_fib_init(double *A, const uint8_t *__restrict__ freev, int HW, int NA, double v0) {
    const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (i < (long long)HW * NA) A[i] = freev[i % HW] ? v0 : 0.0;
}

// ---- value iteration (fp64 Jacobi, reading R24) -----------------------------------------------
// One sweep: V_out(x) = max_a [R(x,a) + gamma (p_int V(t_a) + p_stay V(x) + p_lat (V(t_l1) +
// V(t_l2)))], t_k = N_k(x) if free else x (clamped T); stay: R + gamma V(x).
// The sweep is a no-op once the previous sweep's residual fell below eps, so sweeps can be
// launched in batches without overshooting the oracle's stop rule.
template <uint32_t MASK>
__device__ __forceinline__ double vi_q(const double *__restrict__ V, const double *__restrict__ R64, int HW, int W,
                                       int x, int m8, double p_int, double p_stay, double p_lat, double gamma,
                                       int j) {
    const int k = mask_action(MASK, j);
    double vx = V[x];
    double s;
    if (k == 4) {
        s = vx;
    } else {
        const int l1 = lat1(k), l2 = lat2(k);
        auto tap = [&](int kk) -> double {
            if ((m8 >> nbit(kk)) & 1) return vx;
            return V[x + st_dr(kk) * W + st_dc(kk)];
        };
        s = p_int * tap(k) + p_stay * vx + p_lat * (tap(l1) + tap(l2));
    }
    return R64[(size_t)j * HW + x] + gamma * s;
}

template <uint32_t MASK>
__global__ void k_vi_sweep(const double *__restrict__ Vin, double *__restrict__ Vout,
                           const double *__restrict__ R64, const uint8_t *__restrict__ m8v,
                           const uint8_t *__restrict__ freev, int HW, int W, double p_int, double p_stay,
                           double p_lat, double gamma, unsigned long long *resid, int k, double eps) {
    if (k > 0 && __longlong_as_double((long long)resid[k - 1]) < eps) return;   // converged
    constexpr int NA = mask_count(MASK);
    int x = blockIdx.x * blockDim.x + threadIdx.x;
    double diff = 0.0;
    if (x < HW) {
        double best = 0.0;
        if (freev[x]) {
            int m8 = m8v[x];
            best = -INFINITY;
#pragma unroll
            for (int j = 0; j < NA; ++j) best = fmax(best, vi_q<MASK>(Vin, R64, HW, W, x, m8, p_int, p_stay, p_lat, gamma, j));
        }
        Vout[x] = best;
        diff = fabs(best - Vin[x]);
    }
    for (int o = 16; o > 0; o >>= 1) diff = fmax(diff, __shfl_xor_sync(0xffffffffu, diff, o));
    if ((threadIdx.x & 31) == 0 && diff > 0.0)
        atomicMax(&resid[k], (unsigned long long)__double_as_longlong(diff));   // order-free max
}

template <uint32_t MASK>
__global__ void k_vi_q(const double *__restrict__ V, double *__restrict__ Q64, const double *__restrict__ R64,
                       const uint8_t *__restrict__ m8v, const uint8_t *__restrict__ freev, int HW, int W,
                       double p_int, double p_stay, double p_lat, double gamma) {
    constexpr int NA = mask_count(MASK);
    int x = blockIdx.x * blockDim.x + threadIdx.x;
    if (x >= HW) return;
    int m8 = m8v[x];
#pragma unroll
    for (int j = 0; j < NA; ++j)
        Q64[(size_t)j * HW + x] = freev[x] ? vi_q<MASK>(V, R64, HW, W, x, m8, p_int, p_stay, p_lat, gamma, j) : 0.0;
}

}  // namespace qvts

using namespace qvts;

extern "C" const char *qvts_last_error(void) { return g_last_error.c_str(); }

extern "C" qvts_status qvts_model_create(const qvts_model_desc *d, qvts_model **out) {
    if (!out) { set_error("out is NULL"); return QVTS_ERR_INVALID_ARG; }
    *out = nullptr;
    if (!d || !d->occupancy) { set_error("desc or occupancy is NULL"); return QVTS_ERR_INVALID_ARG; }
    const int H = d->height, W = d->width;
    if (H <= 0 || W <= 0 || (long long)H * W > (1LL << 22)) { set_error("bad grid size"); return QVTS_ERR_INVALID_MODEL; }
    if (d->goal < 0 || d->goal >= H * W || d->occupancy[d->goal]) { set_error("goal must be a free cell"); return QVTS_ERR_INVALID_MODEL; }
    if (d->p_intended < 0 || d->p_stay < 0 || d->p_lateral < 0 ||
        std::fabs(d->p_intended + d->p_stay + 2 * d->p_lateral - 1.0) > 1e-9) {
        set_error("motion noise must satisfy p_int + p_stay + 2 p_lat = 1"); return QVTS_ERR_INVALID_MODEL;
    }
    if (!(d->sensor_acc > 0.5 && d->sensor_acc <= 1.0)) { set_error("sensor_acc must be in (0.5, 1]"); return QVTS_ERR_INVALID_MODEL; }
    if (!(d->gamma > 0.0 && d->gamma < 1.0)) { set_error("gamma must be in (0, 1)"); return QVTS_ERR_INVALID_MODEL; }
    uint32_t mask = d->action_mask & 0x1FF;
    if (mask != 0x1FF && mask != 0x1EF && mask != 0x0AA) {
        set_error("action_mask must be 0x1FF, 0x1EF or 0x0AA"); return QVTS_ERR_INVALID_ARG;
    }
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || d->device < 0 || d->device >= ndev) {
        cudaGetLastError();
        set_error("CUDA device not available"); return QVTS_ERR_CUDA;
    }
    QVTS_CUDA(cudaSetDevice(d->device));

    qvts_model *m = new qvts_model();
    m->device = d->device;
    m->H = H; m->W = W; m->HW = H * W; m->HWp = (H * W + 3) & ~3; m->goal = d->goal; m->mask = mask;
    m->p_int = d->p_intended; m->p_stay = d->p_stay; m->p_lat = d->p_lateral; m->acc = d->sensor_acc;
    m->gamma = d->gamma;
    for (int k = 0; k < 9; ++k) if (mask & (1u << k)) m->action_id[m->NA++] = k;
    m->NAP = (m->NA + 3) & ~3;
    const int HW = m->HW, NA = m->NA;
    m->occ.assign(d->occupancy, d->occupancy + HW);
    for (auto &o : m->occ) o = o ? 1 : 0;
    auto occ_at = [&](int r, int c) -> int {
        if (r < 0 || r >= H || c < 0 || c >= W) return 1;       // off-map = occupied (R4)
        return m->occ[r * W + c];
    };
    m->m8.assign(HW, 0);
    m->sig.assign(HW, 0);
    for (int x = 0; x < HW; ++x) {
        int r = x / W, c = x % W, b = 0;
        for (int k = 0; k < 9; ++k) {
            if (k == 4) continue;
            if (occ_at(r + st_dr(k), c + st_dc(k))) b |= 1 << nbit(k);
        }
        m->m8[x] = (uint8_t)b;
        // wall signature, bit k <-> N_{2k+1} (R6)
        m->sig[x] = (uint8_t)(occ_at(r - 1, c) | (occ_at(r, c - 1) << 1) | (occ_at(r, c + 1) << 2) | (occ_at(r + 1, c) << 3));
    }
    // Reward (R22): pre-clamp T', off-map counts as occupied.
    m->R64.assign((size_t)NA * HW, 0.0);
    for (int x = 0; x < HW; ++x) {
        if (m->occ[x]) continue;
        int r = x / W, c = x % W;
        for (int j = 0; j < NA; ++j) {
            int k = m->action_id[j];
            double v;
            if (k == 4) v = (x == m->goal) ? 0.0 : -2.0;
            else {
                auto rr = [&](int kk) -> double {
                    if (kk == 4) return x == m->goal ? 0.0 : -1.0;
                    int y_r = r + st_dr(kk), y_c = c + st_dc(kk);
                    if (occ_at(y_r, y_c)) return -2.0;
                    return (y_r * W + y_c == m->goal) ? 0.0 : -1.0;
                };
                v = m->p_int * rr(k) + m->p_stay * rr(4) + m->p_lat * (rr(lat1(k)) + rr(lat2(k)));
            }
            m->R64[(size_t)j * HW + x] = v;
        }
    }
    // Stay coefficient of the clamped gather, by neighbour-occupancy byte:
    // c_a(m8) = p_stay + p_int occ(N_a) + p_lat (occ(N_l1) + occ(N_l2)); stay: 1.
    std::vector<float> ctab(256 * m->NAP, 0.f);
    for (int b = 0; b < 256; ++b)
        for (int j = 0; j < NA; ++j) {
            int k = m->action_id[j];
            double c = 1.0;
            if (k != 4)
                c = m->p_stay + m->p_int * ((b >> nbit(k)) & 1) +
                    m->p_lat * (((b >> nbit(lat1(k))) & 1) + ((b >> nbit(lat2(k))) & 1));
            ctab[b * m->NAP + j] = (float)c;
        }
    // O by signature: acc^(4-h) (1-acc)^h, h = popcount(z xor s) (R7).
    std::vector<double> O64(256);
    std::vector<float> O32(256);
    for (int s = 0; s < 16; ++s)
        for (int z = 0; z < 16; ++z) {
            double o = 1.0;
            for (int k = 0; k < 4; ++k) o *= (((s >> k) & 1) == ((z >> k) & 1)) ? m->acc : 1.0 - m->acc;
            O64[s * 16 + z] = o;
            O32[s * 16 + z] = (float)o;
        }
    // Goal terms of R(b,a) = (p_stay - 1) sum b - sum c_a b + sum_x G(x,a) b(x), where
    // G(x,a) = sum_k T'(x,a,k) [N_k(x) = goal] is non-zero only around the goal.
    // Entries grouped by action (action-major, cells in raster order within an action): k_reduce's
    // warp for action j reads [gc_off[j], gc_off[j+1]), at most 9 entries (the goal's 3x3 block).
    std::vector<int32_t> gc_cell, gc_off;
    std::vector<double> gc_val;
    {
        int gr = m->goal / W, gcc = m->goal % W;
        for (int j = 0; j < NA; ++j) {
            gc_off.push_back((int32_t)gc_cell.size());
            const int k = m->action_id[j];
            if (k == 4) continue;
            for (int dr = -1; dr <= 1; ++dr)
                for (int dc = -1; dc <= 1; ++dc) {
                    int r = gr + dr, c = gcc + dc;
                    if (r < 0 || r >= H || c < 0 || c >= W || m->occ[r * W + c]) continue;
                    int x = r * W + c;
                    double g = 0.0;
                    auto hit = [&](int kk) { return (kk == 4) ? (x == m->goal) : (r + st_dr(kk) == gr && c + st_dc(kk) == gcc); };
                    if (hit(k)) g += m->p_int;
                    if (hit(4)) g += m->p_stay;
                    if (hit(lat1(k))) g += m->p_lat;
                    if (hit(lat2(k))) g += m->p_lat;
                    if (g != 0.0) { gc_cell.push_back(x); gc_val.push_back(g); }
                }
        }
        gc_off.push_back((int32_t)gc_cell.size());
    }
    m->ngc = (int)gc_cell.size();
    m->n_free = 0;
    for (int x = 0; x < HW; ++x) m->n_free += m->occ[x] ? 0 : 1;
    std::vector<uint8_t> freev(HW), cell(HW);
    for (int x = 0; x < HW; ++x) {
        freev[x] = m->occ[x] ? 0 : 1;
        cell[x] = (uint8_t)(m->sig[x] | (m->occ[x] << 4));
    }

    qvts_status st = QVTS_OK;
    do {
        if ((st = upload(m->d_m8, m->m8)) != QVTS_OK) break;
        if ((st = upload(m->d_sig, m->sig)) != QVTS_OK) break;
        if ((st = upload(m->d_free, freev)) != QVTS_OK) break;
        if ((st = upload(m->d_cell, cell)) != QVTS_OK) break;
        if ((st = upload(m->d_ctab, ctab)) != QVTS_OK) break;
        if ((st = upload(m->d_R64, m->R64)) != QVTS_OK) break;
        if ((st = upload(m->d_O64, O64)) != QVTS_OK) break;
        if ((st = upload(m->d_O32, O32)) != QVTS_OK) break;
        if ((st = upload(m->d_gc_cell, gc_cell)) != QVTS_OK) break;
        if ((st = upload(m->d_gc_off, gc_off)) != QVTS_OK) break;
        if ((st = upload(m->d_gc_val, gc_val)) != QVTS_OK) break;
        // band sets: ~16K cells per band for many parents, ~2K for few (more CTAs per parent)
        // big bands: as tall as two CTAs' tiles per SM allow, balanced over the grid
        // (QVTS_BAND_ROWS overrides the row count for tuning experiments)
        const int TWp = (W + 5 + 3) & ~3;
        const int max_rows = std::max(1, (int)(100000 / ((long long)TWp * 8)) - 5);
        const int nb_big = (H + max_rows - 1) / max_rows;
        int big_rows = (H + nb_big - 1) / nb_big;
        if (const char *ev = std::getenv("QVTS_BAND_ROWS")) big_rows = std::max(1, std::atoi(ev));
        if ((st = build_bands(*m, m->band_big, big_rows)) != QVTS_OK) break;
        if ((st = build_bands(*m, m->band_small, std::max(1, 1024 / W))) != QVTS_OK) break;
        if ((st = build_leaf_bands(*m, m->leafb)) != QVTS_OK) break;
        if ((st = build_leaf_mma(*m)) != QVTS_OK) break;
        if (cudaEventCreate(&m->ev0) != cudaSuccess || cudaEventCreate(&m->ev1) != cudaSuccess) {
            set_error("cudaEventCreate failed"); st = QVTS_ERR_CUDA; break;
        }
    } while (0);
    if (st != QVTS_OK) { qvts_model_destroy(m); return st; }
    *out = m;
    return QVTS_OK;
}

extern "C" void qvts_model_destroy(qvts_model *m) {
    if (!m) return;
    cudaSetDevice(m->device);
    DevBuf *bufs[] = {&m->d_m8, &m->d_sig, &m->d_cell, &m->bu_R, &m->bu_P, &m->bu_cnt, &m->bu_umask,
                      &m->bu_U, &m->bu_off, &m->bu_path, &m->bu_root, &m->d_ctab, &m->d_R64, &m->d_O64, &m->d_O32, &m->d_gc_cell,
                      &m->d_gc_off, &m->d_gc_val, &m->d_free, &m->d_V[0], &m->d_V[1], &m->d_A[0], &m->d_A[1], &m->d_alpha64, &m->d_resid,
                      &m->d_Q64, &m->part, &m->xs, &m->scan_tmp, &m->total, &m->counters, &m->vshard,
                      &m->ep_b[0], &m->ep_b[1], &m->ep_state, &m->ep_root_step, &m->ep_root_ep,
                      &m->pb_b0, &m->pb_B, &m->pb_G, &m->pb_Gn, &m->pb_GT, &m->pb_Bbar, &m->pb_Sc, &m->pb_Rb,
                      &m->pb_sel, &m->pb_astar, &m->pb_cand, &m->pb_misc, &m->pb_cls, &m->pb_chunks, &m->pb_part};
    for (DevBuf *b : bufs) b->release();
    m->bu_host.release();
    for (DevBuf *b : {&m->lm.wr, &m->lm.offs, &m->lm.dmask, &m->lm.cells, &m->lm.qfr, &m->lm.qfr_fib})
        b->release();
    for (BandSet *bs : {&m->band_big, &m->band_small}) {
        bs->bands.release(); bs->entries.release(); bs->slot_cell.release(); bs->qlist.release(); bs->qlist_fib.release();
    }
    m->leafb.bands.release(); m->leafb.entries.release(); m->leafb.slot_cell.release();
    m->leafb.qlist.release(); m->leafb.qlist_fib.release();
    for (cudaEvent_t e : m->evpool) cudaEventDestroy(e);
    for (auto &v : m->vl) { v.path.release(); v.parent_q.release(); v.z.release(); v.f.release(); v.root.release(); v.V.release(); v.belief.release(); }
    for (DevBuf *b : {&m->bf_bel, &m->bf_path, &m->bf_pq, &m->bf_z, &m->bf_f, &m->bf_root, &m->bf_depth, &m->bf_vU,
                      &m->bf_vL, &m->bf_vH, &m->bf_vE, &m->bf_vq0, &m->bf_vLa, &m->bf_qR, &m->bf_qU, &m->bf_qL,
                      &m->bf_qH, &m->bf_qE, &m->bf_qc0, &m->bf_qnc, &m->bf_qv, &m->bf_VT, &m->bf_part, &m->bf_sum,
                      &m->bf_keys, &m->bf_anc, &m->bf_rtr})
        b->release();
    {
        QLevel &q = m->bf_ql;
        q.vmap.release(); q.R.release(); q.P.release(); q.cnt.release(); q.umask.release(); q.U.release();
        q.off.release(); q.Q.release(); q.zdraw.release(); q.leafV.release();
    }
    for (auto &q : m->ql) { q.vmap.release(); q.R.release(); q.P.release(); q.cnt.release(); q.umask.release(); q.U.release(); q.off.release(); q.Q.release(); q.zdraw.release(); q.leafV.release(); q.xdraw.release(); }
    if (m->bf_gexec) cudaGraphExecDestroy(m->bf_gexec);
    if (m->pg_exec) cudaGraphExecDestroy(m->pg_exec);
    if (m->pg_stream) cudaStreamDestroy(m->pg_stream);
    if (m->pg_join) cudaEventDestroy(m->pg_join);
    m->lvl_cnt.release();
    m->root_buf.release();
    if (m->bf_stream) cudaStreamDestroy(m->bf_stream);
    if (m->bf_join) cudaEventDestroy(m->bf_join);
    if (m->ev0) cudaEventDestroy(m->ev0);
    if (m->ev1) cudaEventDestroy(m->ev1);
    delete m;
}

extern "C" qvts_status qvts_set_profiling(qvts_model *m, int32_t enable) {
    if (!m) { set_error("model is NULL"); return QVTS_ERR_INVALID_ARG; }
    m->prof = enable != 0;
    m->pstat = qvts_profile{};
    m->evrecs.clear();
    m->evnext = 0;
    return QVTS_OK;
}

extern "C" qvts_status qvts_get_profile(const qvts_model *m, qvts_profile *out) {
    if (!m || !out) { set_error("NULL argument"); return QVTS_ERR_INVALID_ARG; }
    *out = m->pstat;
    return QVTS_OK;
}

extern "C" qvts_status qvts_model_info(const qvts_model *m, int32_t *n_actions, int32_t *action_ids, int64_t *n_cells) {
    if (!m) { set_error("model is NULL"); return QVTS_ERR_INVALID_ARG; }
    if (n_actions) *n_actions = m->NA;
    if (action_ids) for (int j = 0; j < 9; ++j) action_ids[j] = j < m->NA ? m->action_id[j] : -1;
    if (n_cells) *n_cells = m->HW;
    return QVTS_OK;
}

extern "C" qvts_status qvts_model_tables(const qvts_model *m, float *R_host, uint8_t *sig_host) {
    if (!m) { set_error("model is NULL"); return QVTS_ERR_INVALID_ARG; }
    if (R_host) for (size_t i = 0; i < m->R64.size(); ++i) R_host[i] = (float)m->R64[i];
    if (sig_host) std::memcpy(sig_host, m->sig.data(), m->HW);
    return QVTS_OK;
}

extern "C" qvts_status qvts_value_iteration(qvts_model *m, double eps, int32_t max_sweeps, int32_t *sweeps_out,
                                            double *residual_out, void *stream) {
    qvts::NvtxRange nvtx_range__("qvts_value_iteration");
    if (!m || !(eps > 0) || max_sweeps <= 0) { set_error("bad value_iteration arguments"); return QVTS_ERR_INVALID_ARG; }
    QVTS_CUDA(cudaSetDevice(m->device));
    cudaStream_t st = (cudaStream_t)stream;
    const int HW = m->HW, NA = m->NA;
    QVTS_TRY(m->d_V[0].ensure(sizeof(double) * HW));
    QVTS_TRY(m->d_V[1].ensure(sizeof(double) * HW));
    QVTS_TRY(m->d_resid.ensure(sizeof(unsigned long long) * (size_t)max_sweeps));
    QVTS_TRY(m->d_Q64.ensure(sizeof(double) * (size_t)NA * HW));
    QVTS_CUDA(cudaMemsetAsync(m->d_V[0].p, 0, sizeof(double) * HW, st));
    QVTS_CUDA(cudaMemsetAsync(m->d_resid.p, 0, sizeof(unsigned long long) * (size_t)max_sweeps, st));
    const int blk = 256, grid = (HW + blk - 1) / blk;
    std::vector<unsigned long long> res(max_sweeps);
    int done = -1, k = 0;
    const int batch = 32;
    while (k < max_sweeps && done < 0) {
        int k1 = std::min(max_sweeps, k + batch);
        for (int kk = k; kk < k1; ++kk) {
            const double *vin = m->d_V[kk & 1].as<double>();
            double *vout = m->d_V[(kk + 1) & 1].as<double>();
#define QVTS_VI_LAUNCH(MASK)                                                                              \
    k_vi_sweep<MASK><<<grid, blk, 0, st>>>(vin, vout, m->d_R64.as<double>(), m->d_m8.as<uint8_t>(),       \
                                           m->d_free.as<uint8_t>(), HW, m->W, m->p_int, m->p_stay, m->p_lat, \
                                           m->gamma, m->d_resid.as<unsigned long long>(), kk, eps)
            QVTS_DISPATCH_MASK(m->mask, QVTS_VI_LAUNCH);
#undef QVTS_VI_LAUNCH
        }
        QVTS_CUDA(cudaGetLastError());
        QVTS_CUDA(cudaMemcpyAsync(res.data() + k, m->d_resid.as<unsigned long long>() + k,
                                  sizeof(unsigned long long) * (k1 - k), cudaMemcpyDeviceToHost, st));
        QVTS_CUDA(cudaStreamSynchronize(st));
        for (int kk = k; kk < k1; ++kk) {
            double r;
            std::memcpy(&r, &res[kk], sizeof(double));
            if (r < eps) { done = kk; break; }
        }
        k = k1;
    }
    int last = done >= 0 ? done : max_sweeps - 1;
    double resid;
    std::memcpy(&resid, &res[last], sizeof(double));
    const double *vfinal = m->d_V[(last + 1) & 1].as<double>();
#define QVTS_VIQ_LAUNCH(MASK)                                                                          \
    k_vi_q<MASK><<<grid, blk, 0, st>>>(vfinal, m->d_Q64.as<double>(), m->d_R64.as<double>(),          \
                                       m->d_m8.as<uint8_t>(), m->d_free.as<uint8_t>(), HW, m->W, m->p_int, \
                                       m->p_stay, m->p_lat, m->gamma)
    QVTS_DISPATCH_MASK(m->mask, QVTS_VIQ_LAUNCH);
#undef QVTS_VIQ_LAUNCH
    QVTS_CUDA(cudaGetLastError());
    // leaf offset qbar = midpoint of the Q range on free cells (SURVEY c.6 rule 5)
    std::vector<double> V(HW);
    QVTS_CUDA(cudaMemcpyAsync(V.data(), vfinal, sizeof(double) * HW, cudaMemcpyDeviceToHost, st));
    QVTS_CUDA(cudaStreamSynchronize(st));
    double lo = INFINITY, hi = -INFINITY;
    for (int x = 0; x < HW; ++x)
        if (!m->occ[x]) { lo = std::min(lo, V[x]); hi = std::max(hi, V[x]); }
    m->qbar = std::isfinite(lo) ? 0.5 * (lo + hi) : 0.0;
    QVTS_TRY(build_qlists(*m, m->d_Q64.as<double>(), m->qbar, false, st));
    QVTS_CUDA(cudaStreamSynchronize(st));
    m->have_q = true;
    if (sweeps_out) *sweeps_out = last + 1;
    if (residual_out) *residual_out = resid;
    if (done < 0) { set_error("value iteration did not converge"); return QVTS_ERR_NOT_CONVERGED; }
    return QVTS_OK;
}

extern "C" qvts_status qvts_fib_iteration(qvts_model *m, double eps, int32_t max_sweeps, int32_t *sweeps_out,
                                          double *residual_out, void *stream) {
    qvts::NvtxRange nvtx_range__("qvts_fib_iteration");
    if (!m || !(eps > 0) || max_sweeps <= 0) { set_error("bad fib_iteration arguments"); return QVTS_ERR_INVALID_ARG; }
    QVTS_CUDA(cudaSetDevice(m->device));
    cudaStream_t st = (cudaStream_t)stream;
    const int HW = m->HW, NA = m->NA;
    const size_t nA = (size_t)NA * HW;
    QVTS_TRY(m->d_A[0].ensure(sizeof(double) * nA));
    QVTS_TRY(m->d_A[1].ensure(sizeof(double) * nA));
    QVTS_TRY(m->d_alpha64.ensure(sizeof(double) * nA));
    QVTS_TRY(m->d_resid.ensure(sizeof(unsigned long long) * (size_t)max_sweeps));
    QVTS_CUDA(cudaMemsetAsync(m->d_resid.p, 0, sizeof(unsigned long long) * (size_t)max_sweeps, st));
    double rmax = -INFINITY;
    for (size_t i = 0; i < m->R64.size(); ++i)
        if (!m->occ[i % HW]) rmax = std::max(rmax, m->R64[i]);
    k_fib_init<<<(unsigned)((nA + 255) / 256), 256, 0, st>>>(m->d_A[0].as<double>(), m->d_free.as<uint8_t>(), HW, NA,
                                                            rmax / (1.0 - m->gamma));
    QVTS_CUDA(cudaGetLastError());
    const int blk = 128, grid = (HW + blk - 1) / blk;
    std::vector<unsigned long long> res(max_sweeps);
    int done = -1, k = 0;
    while (k < max_sweeps && done < 0) {
        const int k1 = std::min(max_sweeps, k + 32);
        for (int kk = k; kk < k1; ++kk) {
#define QVTS_FIB_LAUNCH(MASK)                                                                                    \
    k_fib_sweep<MASK><<<grid, blk, 0, st>>>(m->d_A[kk & 1].as<double>(), m->d_A[(kk + 1) & 1].as<double>(),       \
                                            m->d_R64.as<double>(), m->d_m8.as<uint8_t>(), m->d_free.as<uint8_t>(), \
                                            m->d_sig.as<uint8_t>(), m->d_O64.as<double>(), HW, m->W, m->p_int,     \
                                            m->p_stay, m->p_lat, m->gamma, m->d_resid.as<unsigned long long>(), kk, eps)
            QVTS_DISPATCH_MASK(m->mask, QVTS_FIB_LAUNCH);
#undef QVTS_FIB_LAUNCH
        }
        QVTS_CUDA(cudaGetLastError());
        QVTS_CUDA(cudaMemcpyAsync(res.data() + k, m->d_resid.as<unsigned long long>() + k,
                                  sizeof(unsigned long long) * (k1 - k), cudaMemcpyDeviceToHost, st));
        QVTS_CUDA(cudaStreamSynchronize(st));
        for (int kk = k; kk < k1; ++kk) {
            double r;
            std::memcpy(&r, &res[kk], sizeof(double));
            if (r < eps) { done = kk; break; }
        }
        k = k1;
    }
    const int last = done >= 0 ? done : max_sweeps - 1;
    double resid;
    std::memcpy(&resid, &res[last], sizeof(double));
    QVTS_CUDA(cudaMemcpyAsync(m->d_alpha64.p, m->d_A[(last + 1) & 1].p, sizeof(double) * nA, cudaMemcpyDeviceToDevice, st));
    std::vector<double> A(nA);
    QVTS_CUDA(cudaMemcpyAsync(A.data(), m->d_alpha64.p, sizeof(double) * nA, cudaMemcpyDeviceToHost, st));
    QVTS_CUDA(cudaStreamSynchronize(st));
    double lo = INFINITY, hi = -INFINITY;
    for (size_t i = 0; i < nA; ++i)
        if (!m->occ[i % HW]) { lo = std::min(lo, A[i]); hi = std::max(hi, A[i]); }
    m->qbar_fib = std::isfinite(lo) ? 0.5 * (lo + hi) : 0.0;
    QVTS_TRY(build_qlists(*m, m->d_alpha64.as<double>(), m->qbar_fib, true, st));
    QVTS_CUDA(cudaStreamSynchronize(st));
    m->have_fib = true;
    if (sweeps_out) *sweeps_out = last + 1;
    if (residual_out) *residual_out = resid;
    if (done < 0) { set_error("FIB iteration did not converge"); return QVTS_ERR_NOT_CONVERGED; }
    return QVTS_OK;
}

extern "C" qvts_status qvts_get_alpha(const qvts_model *m, double *alpha_host) {
    if (!m || !alpha_host) { set_error("NULL argument"); return QVTS_ERR_INVALID_ARG; }
    if (!m->have_fib) { set_error("FIB iteration has not run"); return QVTS_ERR_STATE; }
    QVTS_CUDA(cudaSetDevice(m->device));
    QVTS_CUDA(cudaMemcpy(alpha_host, m->d_alpha64.p, sizeof(double) * (size_t)m->NA * m->HW, cudaMemcpyDeviceToHost));
    return QVTS_OK;
}

extern "C" qvts_status qvts_get_q(const qvts_model *m, double *q_host) {
    if (!m || !q_host) { set_error("NULL argument"); return QVTS_ERR_INVALID_ARG; }
    if (!m->have_q) { set_error("value iteration has not run"); return QVTS_ERR_STATE; }
    QVTS_CUDA(cudaSetDevice(m->device));
    QVTS_CUDA(cudaMemcpy(q_host, m->d_Q64.p, sizeof(double) * (size_t)m->NA * m->HW, cudaMemcpyDeviceToHost));
    return QVTS_OK;
}
