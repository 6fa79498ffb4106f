// episodes.cu — qvts_run_episodes: the closed-loop outer loop of Alg. 1
// over a batch of episodes at once.  Per step, all active episodes are planned
// together (their beliefs are the roots of one level-batched plan, in memory-sized waves), then
// k_env draws the true motion and the observation from Philox environment streams, accumulates
// the discounted return (Eq. 1) and the stop streak (readings R26/R27), and the belief of every
// episode is advanced with Eq. 3 using the marginals the plan already computed at its root.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <queue>
#include <vector>

#include "philox.cuh"
#include "qvts_internal.cuh"
#include "stencil.cuh"

namespace qvts {

struct EpArgs {
    int n_owned;
    int32_t *ep_id, *x, *x0, *streak, *steps, *collisions, *outcome, *aidx, *act;
    double *ret, *disc;
};

// fp64 prefix sums of the initial belief (inverse-CDF table for x0 ~ b0, Appendix A.5)
__global__ void __launch_bounds__(1024) k_cdf(const float *__restrict__ b0, double *__restrict__ cdf, int n) {
    __shared__ double wsum[32];
    __shared__ double carry_s;
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
    if (t == 0) carry_s = 0.0;
    __syncthreads();
    for (int base = 0; base < n; base += 1024) {
        const int i = base + t;
        const double v = i < n ? (double)b0[i] : 0.0;
        double s = v;
        for (int o = 1; o < 32; o <<= 1) {
            const double y = __shfl_up_sync(0xffffffffu, s, o);
            if (lane >= o) s += y;
        }
        if (lane == 31) wsum[warp] = s;
        __syncthreads();
        if (warp == 0) {
            double ws = wsum[lane];
            for (int o = 1; o < 32; o <<= 1) {
                const double y = __shfl_up_sync(0xffffffffu, ws, o);
                if (lane >= o) ws += y;
            }
            wsum[lane] = ws;
        }
        __syncthreads();
        const double carry = carry_s;
        if (i < n) cdf[i] = carry + (warp ? wsum[warp - 1] : 0.0) + s;
        __syncthreads();
        if (t == 1023) carry_s = carry + wsum[31];
        __syncthreads();
    }
}

__global__ void k_uniform_b0(const uint8_t *__restrict__ freev, int HW, float inv, float *__restrict__ b0) {
    const int x = blockIdx.x * blockDim.x + threadIdx.x;
    if (x < HW) b0[x] = freev[x] ? inv : 0.f;
}

// x0 ~ b0 with word 2 of the step-0 environment draw; every slot starts from b0
__global__ void k_ep_init(EpArgs e, const double *__restrict__ cdf, int HW, uint32_t seed,
                          const float *__restrict__ b0, float *__restrict__ bel, long long stride) {
    const int i = blockIdx.x;
    if (i >= e.n_owned) return;
    for (int x = threadIdx.x; x < HW; x += blockDim.x) bel[(long long)i * stride + x] = b0[x];
    if (threadIdx.x == 0) {
        const uint4 r = philox4x32_10(make_uint4(0u, 0u, 0u, 0u), make_uint2(seed, (uint32_t)e.ep_id[i]));
        const double tt = philox_uniform(r.z) * cdf[HW - 1];
        int lo = 0, hi = HW - 1;                     // min{k : tt < C_k}
        while (lo < hi) {
            const int mid = (lo + hi) >> 1;
            if (tt < cdf[mid]) hi = mid; else lo = mid + 1;
        }
        e.x[i] = lo; e.x0[i] = lo;
        e.streak[i] = 0; e.steps[i] = 0; e.collisions[i] = 0; e.outcome[i] = -1;
        e.ret[i] = 0.0; e.disc[i] = 1.0;
    }
}

__global__ void k_fill_u32(uint32_t *p, int n, uint32_t v) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) p[i] = v;
}
__global__ void k_copy_i32_u32(const int32_t *src, uint32_t *dst, int n) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) dst[i] = (uint32_t)src[i];
}

// QVTS action = argmax_a Q(root, a), ties -> lowest stencil id (R16/R18)
__global__ void k_pick_qvts(EpArgs e, const int32_t *__restrict__ active, int nw, const double *__restrict__ Q,
                            int NA, const int32_t *__restrict__ act_ids) {
    const int w = blockIdx.x * blockDim.x + threadIdx.x;
    if (w >= nw) return;
    int best = 0;
    for (int j = 1; j < NA; ++j)
        if (Q[(long long)w * NA + j] > Q[(long long)w * NA + best]) best = j;
    const int i = active[w];
    e.aidx[i] = best;
    e.act[i] = act_ids[best];
}

// belief mode (argmax, ties -> lowest index, R30): one block per episode
__global__ void __launch_bounds__(256) k_mode(const int32_t *__restrict__ active, const float *__restrict__ bel,
                                              long long stride, int HW, int32_t *__restrict__ mode) {
    const int w = blockIdx.x;
    const int i = active[w];
    const float *b = bel + (long long)i * stride;
    float bv = -1.f;
    int bi = 0x7fffffff;
    for (int x = threadIdx.x; x < HW; x += blockDim.x) {
        const float v = b[x];
        if (v > bv) { bv = v; bi = x; }
    }
    __shared__ float sv[256];
    __shared__ int si[256];
    sv[threadIdx.x] = bv;
    si[threadIdx.x] = bi;
    __syncthreads();
    for (int o = 128; o > 0; o >>= 1) {
        if (threadIdx.x < o) {
            const float v2 = sv[threadIdx.x + o];
            const int i2 = si[threadIdx.x + o];
            if (v2 > sv[threadIdx.x] || (v2 == sv[threadIdx.x] && i2 < si[threadIdx.x])) {
                sv[threadIdx.x] = v2;
                si[threadIdx.x] = i2;
            }
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) mode[w] = si[0];
}

// MDP baseline: one table lookup at the belief mode
__global__ void k_pick_mdp(EpArgs e, const int32_t *__restrict__ active, int nw, const int32_t *__restrict__ mode,
                           const double *__restrict__ Q64, int NA, int HW, const int32_t *__restrict__ act_ids) {
    const int w = blockIdx.x * blockDim.x + threadIdx.x;
    if (w >= nw) return;
    const int xm = mode[w];
    int best = 0;
    for (int j = 1; j < NA; ++j)
        if (Q64[(long long)j * HW + xm] > Q64[(long long)best * HW + xm]) best = j;
    const int i = active[w];
    e.aidx[i] = best;
    e.act[i] = act_ids[best];
}

__global__ void k_set_actions(EpArgs e, const int32_t *__restrict__ active, int nw, const int32_t *__restrict__ aidx,
                              const int32_t *__restrict__ act_ids) {
    const int w = blockIdx.x * blockDim.x + threadIdx.x;
    if (w >= nw) return;
    const int i = active[w];
    e.aidx[i] = aidx[w];
    e.act[i] = act_ids[aidx[w]];
}

struct EnvArgs {
    int H, W, NA, goal, max_steps, patience;
    double p_int, p_stay, p_lat, acc, gamma;
    uint32_t seed;
    const uint8_t *occ, *sig;
    const double *R64;       // [NA][HW]
    const double *P;         // plan / marginal P(z|b,a) of the wave, [w][NA][16]
    int32_t *sel_q, *sel_z, *sel_out;
    int32_t *log_a, *log_z, *log_x;   // [n_owned][max_steps] or NULL
};

// One environment step per active episode: y ~ T'(x,a,.) in stencil order (an occupied or
// off-map y is a collision and the robot stays), z ~ O(x',.), return += gamma^s
// R(x,a) (Eq. 1, R27), stop streak and step cap (R26).  Word 0 drives motion, word 1 sensing.
__global__ void k_env(EpArgs e, EnvArgs v, const int32_t *__restrict__ active, int nw) {
    const int w = blockIdx.x * blockDim.x + threadIdx.x;
    if (w >= nw) return;
    const int i = active[w];
    const int s = e.steps[i];
    const int x = e.x[i], k = e.act[i], j = e.aidx[i];
    const uint4 r = philox4x32_10(make_uint4(0u, 0u, 0u, (uint32_t)s), make_uint2(v.seed, (uint32_t)e.ep_id[i]));
    // motion: pre-clamp T'(x,a,.) over stencil offsets, fp64 CDF in stencil order
    double wgt[9];
    for (int kk = 0; kk < 9; ++kk) wgt[kk] = 0.0;
    if (k == 4) {
        wgt[4] = 1.0;
    } else {
        wgt[k] += v.p_int;
        wgt[4] += v.p_stay;
        wgt[lat1(k)] += v.p_lat;
        wgt[lat2(k)] += v.p_lat;
    }
    double C[16];
    double acc = 0.0;
    for (int kk = 0; kk < 9; ++kk) { acc += wgt[kk]; C[kk] = acc; }
    double tt = philox_uniform(r.x) * C[8];
    int kd = 8;
    for (int kk = 0; kk < 9; ++kk) if (tt < C[kk]) { kd = kk; break; }
    int xn = x;
    if (kd != 4) {
        const int rr = x / v.W + st_dr(kd), cc = x % v.W + st_dc(kd);
        if (rr < 0 || rr >= v.H || cc < 0 || cc >= v.W || v.occ[rr * v.W + cc]) e.collisions[i] += 1;
        else xn = rr * v.W + cc;
    }
    // observation z ~ O(x',.): product over the 4 independent sensors (R7), fp64
    const int sg = v.sig[xn];
    acc = 0.0;
    for (int z = 0; z < 16; ++z) {
        double o = 1.0;
        for (int b = 0; b < 4; ++b) o *= (((z >> b) & 1) == ((sg >> b) & 1)) ? v.acc : (1.0 - v.acc);
        acc += o;
        C[z] = acc;
    }
    tt = philox_uniform(r.y) * C[15];
    int z = 15;
    for (int zz = 0; zz < 16; ++zz) if (tt < C[zz]) { z = zz; break; }
    e.ret[i] += e.disc[i] * v.R64[(long long)j * v.H * v.W + x];
    e.disc[i] *= v.gamma;
    if (v.log_a) {
        const long long li = (long long)i * v.max_steps + s;
        v.log_a[li] = k; v.log_z[li] = z; v.log_x[li] = xn;
    }
    e.x[i] = xn;
    e.steps[i] = s + 1;
    v.sel_q[w] = w * v.NA + j;
    v.sel_z[w] = z;
    v.sel_out[w] = i;
    if (!(v.P[((long long)w * v.NA + j) * 16 + z] > 1e-30)) { e.outcome[i] = 3; return; }   // Eq. 3 undefined
    e.streak[i] = (k == 4) ? e.streak[i] + 1 : 0;
    if (v.patience > 0 && e.streak[i] >= v.patience) e.outcome[i] = (xn == v.goal) ? 0 : 1;
    else if (s + 1 >= v.max_steps) e.outcome[i] = 2;
}

// next active list (slot order) and its size
__global__ void __launch_bounds__(1024) k_compact(const int32_t *__restrict__ outcome, int n, int32_t *__restrict__ active,
                                                  int32_t *__restrict__ count) {
    __shared__ int wsum[32];
    __shared__ int carry_s;
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
    if (t == 0) carry_s = 0;
    __syncthreads();
    for (int base = 0; base < n; base += 1024) {
        const int i = base + t;
        const int f = (i < n && outcome[i] < 0) ? 1 : 0;
        const unsigned bal = __ballot_sync(0xffffffffu, f);
        if (lane == 0) wsum[warp] = __popc(bal);
        __syncthreads();
        if (warp == 0) {
            int ws = wsum[lane];
            for (int o = 1; o < 32; o <<= 1) {
                const int y = __shfl_up_sync(0xffffffffu, ws, o);
                if (lane >= o) ws += y;
            }
            wsum[lane] = ws;
        }
        __syncthreads();
        const int pos = carry_s + (warp ? wsum[warp - 1] : 0) + __popc(bal & ((1u << lane) - 1u));
        if (f) active[pos] = i;
        __syncthreads();
        if (t == 0) carry_s += wsum[31];
        __syncthreads();
    }
    if (t == 0) *count = carry_s;
}

__global__ void k_records(EpArgs e, double *__restrict__ rec, int n_total) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= e.n_owned) return;
    double *r = rec + (long long)e.ep_id[i] * 6;
    r[0] = e.outcome[i] < 0 ? 2.0 : (double)e.outcome[i];
    r[1] = e.steps[i];
    r[2] = e.collisions[i];
    r[3] = e.x0[i];
    r[4] = e.x[i];
    r[5] = e.ret[i] + 0.0;
    (void)n_total;
}

// ---- A* comparator on the belief mode (reading R29): unit-cost moves of the
// action set, Chebyshev (diagonals) or Manhattan heuristic, priority (f, cell), neighbours in
// ascending stencil id; returns the first move's stencil id, stay at the goal.
static int astar_first_move(const Model &m, int start) {
    if (start == m.goal) return 4;
    const int H = m.H, W = m.W, HW = m.HW;
    bool diag = false;
    for (int j = 0; j < m.NA; ++j) {
        const int k = m.action_id[j];
        if (k != 4 && st_dr(k) != 0 && st_dc(k) != 0) diag = true;
    }
    const int gr = m.goal / W, gc = m.goal % W;
    auto heur = [&](int x) {
        const int dr = std::abs(x / W - gr), dc = std::abs(x % W - gc);
        return diag ? std::max(dr, dc) : dr + dc;
    };
    std::vector<int> g(HW, -1), par(HW, -1);
    std::vector<char> closed(HW, 0);
    using Item = std::pair<long long, int>;
    std::priority_queue<Item, std::vector<Item>, std::greater<Item>> open;
    g[start] = 0;
    open.push({((long long)heur(start) << 32) | start, start});
    bool found = false;
    while (!open.empty()) {
        const int x = open.top().second;
        open.pop();
        if (closed[x]) continue;
        closed[x] = 1;
        if (x == m.goal) { found = true; break; }
        const int r = x / W, c = x % W;
        for (int j = 0; j < m.NA; ++j) {
            const int k = m.action_id[j];
            if (k == 4) continue;
            const int rr = r + st_dr(k), cc = c + st_dc(k);
            if (rr < 0 || rr >= H || cc < 0 || cc >= W) continue;
            const int y = rr * W + cc;
            if (m.occ[y] || closed[y]) continue;
            if (g[y] < 0 || g[x] + 1 < g[y]) {
                g[y] = g[x] + 1;
                par[y] = x;
                open.push({((long long)(g[y] + heur(y)) << 32) | y, y});
            }
        }
    }
    if (!found) return 4;
    int y = m.goal;
    while (par[y] != start) y = par[y];
    return 3 * (y / W - start / W + 1) + (y % W - start % W + 1);
}

}  // namespace qvts

using namespace qvts;

extern "C" qvts_status qvts_run_episodes(qvts_model *m, const qvts_episode_cfg *cfg, const qvts_comm *comm,
                                         qvts_episode_record *out_host, void *stream) {
    qvts::NvtxRange nvtx_range__("qvts_run_episodes");
    if (!m || !cfg || !out_host || cfg->n_episodes < 0 || cfg->max_steps < 1 || cfg->stop_patience < 0 ||
        cfg->planner < 0 || cfg->planner > 2) {
        set_error("bad run_episodes arguments");
        return QVTS_ERR_INVALID_ARG;
    }
    if (cfg->planner == QVTS_PLANNER_QVTS && (cfg->depth < 1 || cfg->depth > 8 || cfg->n_samples < 1 ||
                                              cfg->n_samples > 4096)) {
        set_error("depth must be 1..8 and n_samples 1..4096");
        return QVTS_ERR_INVALID_ARG;
    }
    if (!m->have_q) { set_error("run qvts_value_iteration before episodes"); return QVTS_ERR_STATE; }
    if (comm && (comm->nranks < 1 || comm->rank < 0 || comm->rank >= comm->nranks ||
                 (comm->nranks > 1 && !comm->allreduce_sum_f64))) {
        set_error("bad comm"); return QVTS_ERR_INVALID_ARG;
    }
    QVTS_CUDA(cudaSetDevice(m->device));
    cudaStream_t st = (cudaStream_t)stream;
    const int E = cfg->n_episodes, G = comm ? comm->nranks : 1, rank = comm ? comm->rank : 0;
    const int HW = m->HW, NA = m->NA, MS = cfg->max_steps;
    std::vector<int32_t> owned;
    for (int e = 0; e < E; ++e) if (e % G == rank) owned.push_back(e);
    const int no = (int)owned.size();
    std::memset(out_host, 0, sizeof(qvts_episode_record) * (size_t)E);

    // device state (SoA)
    DevBuf st_i32, st_f64, bel[2], b0buf, cdf, act_ids, act_list, wave_tmp, cnt, recbuf, logs, ukeys;
    auto cleanup = [&]() {
        for (DevBuf *b : {&st_i32, &st_f64, &bel[0], &bel[1], &b0buf, &cdf, &act_ids, &act_list, &wave_tmp, &cnt,
                          &recbuf, &logs, &ukeys})
            b->release();
        // level maps pointing into the released active lists must not outlive them:
        // a later trace accessor would read freed memory
        for (auto &q : m->ql) { q.mapped = false; q.vmap_ptr = nullptr; }
    };
    qvts_status s = QVTS_OK;
    const int nn = std::max(1, no);
    if ((s = st_i32.ensure(sizeof(int32_t) * 9 * nn)) != QVTS_OK ||
        (s = st_f64.ensure(sizeof(double) * 2 * nn)) != QVTS_OK ||
        (s = bel[0].ensure(sizeof(float) * (size_t)nn * m->HWp)) != QVTS_OK ||
        (s = bel[1].ensure(sizeof(float) * (size_t)nn * m->HWp)) != QVTS_OK ||
        (s = b0buf.ensure(sizeof(float) * HW)) != QVTS_OK || (s = cdf.ensure(sizeof(double) * HW)) != QVTS_OK ||
        (s = act_ids.ensure(sizeof(int32_t) * 9)) != QVTS_OK ||
        (s = act_list.ensure(sizeof(int32_t) * nn)) != QVTS_OK ||
        (s = wave_tmp.ensure(sizeof(int32_t) * 4 * nn)) != QVTS_OK || (s = cnt.ensure(sizeof(int32_t))) != QVTS_OK ||
        (s = recbuf.ensure(sizeof(double) * 6 * std::max(1, E))) != QVTS_OK ||
        (s = ukeys.ensure(sizeof(uint32_t) * 2 * nn)) != QVTS_OK) {
        cleanup();
        return s;
    }
    EpArgs ea;
    int32_t *I = st_i32.as<int32_t>();
    ea.n_owned = no;
    ea.ep_id = I; ea.x = I + nn; ea.x0 = I + 2 * nn; ea.streak = I + 3 * nn; ea.steps = I + 4 * nn;
    ea.collisions = I + 5 * nn; ea.outcome = I + 6 * nn; ea.aidx = I + 7 * nn; ea.act = I + 8 * nn;
    ea.ret = st_f64.as<double>(); ea.disc = st_f64.as<double>() + nn;
    uint32_t *root_step = ukeys.as<uint32_t>(), *root_ep = ukeys.as<uint32_t>() + nn;
    int32_t *sel_q = wave_tmp.as<int32_t>(), *sel_z = sel_q + nn, *sel_out = sel_q + 2 * nn, *mode = sel_q + 3 * nn;
    int32_t *log_a = nullptr, *log_z = nullptr, *log_x = nullptr;
    const bool want_log = cfg->log_actions || cfg->log_obs || cfg->log_states;
    if (want_log) {
        if ((s = logs.ensure(sizeof(int32_t) * 3 * (size_t)nn * MS)) != QVTS_OK) { cleanup(); return s; }
        log_a = logs.as<int32_t>(); log_z = log_a + (size_t)nn * MS; log_x = log_z + (size_t)nn * MS;
        QVTS_CUDA(cudaMemsetAsync(logs.p, 0xFF, sizeof(int32_t) * 3 * (size_t)nn * MS, st));
    }
#define EP_CUDA(call)                                                            \
    do {                                                                         \
        cudaError_t e__ = (call);                                                \
        if (e__ != cudaSuccess) {                                                \
            set_error(std::string(#call) + ": " + cudaGetErrorString(e__));      \
            cleanup();                                                           \
            return QVTS_ERR_CUDA;                                                \
        }                                                                        \
    } while (0)
#define EP_TRY(expr)                       \
    do {                                   \
        qvts_status s2 = (expr);           \
        if (s2 != QVTS_OK) { cleanup(); return s2; } \
    } while (0)

    if (no > 0) EP_CUDA(cudaMemcpyAsync(ea.ep_id, owned.data(), sizeof(int32_t) * no, cudaMemcpyHostToDevice, st));
    EP_CUDA(cudaMemcpyAsync(act_ids.p, m->action_id, sizeof(int32_t) * 9, cudaMemcpyHostToDevice, st));
    const float *b0 = cfg->b0_dev;
    if (!b0) {
        k_uniform_b0<<<(HW + 255) / 256, 256, 0, st>>>(m->d_free.as<uint8_t>(), HW, (float)(1.0 / (double)m->n_free),
                                                      b0buf.as<float>());
        b0 = b0buf.as<float>();
    }
    k_cdf<<<1, 1024, 0, st>>>(b0, cdf.as<double>(), HW);
    if (no > 0) {
        k_ep_init<<<no, 256, 0, st>>>(ea, cdf.as<double>(), HW, cfg->seed, b0, bel[0].as<float>(), m->HWp);
        k_copy_i32_u32<<<(no + 255) / 256, 256, 0, st>>>(ea.ep_id, root_ep, no);
        k_compact<<<1, 1024, 0, st>>>(ea.outcome, no, act_list.as<int32_t>(), cnt.as<int32_t>());
    }
    EP_CUDA(cudaGetLastError());

    // plan-wave size from free device memory (beliefs of levels 1..D-1 per root)
    size_t fmem = 0, tmem = 0;
    cudaMemGetInfo(&fmem, &tmem);
    double per_root = 0.0, lvl = 1.0;
    for (int d = 1; d < cfg->depth; ++d) { lvl *= NA * std::min(cfg->n_samples, 6); per_root += lvl; }
    per_root = per_root * m->HWp * 4.0 * 1.25 + 1e6;
    int wave = (int)std::max(1.0, std::min((double)std::max(no, 1), 0.45 * (double)fmem / per_root));
    if (const char *ev = std::getenv("QVTS_EPISODE_WAVE")) wave = std::max(1, std::atoi(ev));

    EnvArgs env;
    env.H = m->H; env.W = m->W; env.NA = NA; env.goal = m->goal; env.max_steps = MS; env.patience = cfg->stop_patience;
    env.p_int = m->p_int; env.p_stay = m->p_stay; env.p_lat = m->p_lat; env.acc = m->acc; env.gamma = m->gamma;
    env.seed = cfg->seed; env.sig = m->d_sig.as<uint8_t>();
    env.R64 = m->d_R64.as<double>(); env.sel_q = sel_q; env.sel_z = sel_z; env.sel_out = sel_out;
    env.log_a = log_a; env.log_z = log_z; env.log_x = log_x;
    // k_env tests occupancy through d_occ: build it once
    DevBuf occb;
    EP_TRY(occb.ensure(HW));
    EP_CUDA(cudaMemcpyAsync(occb.p, m->occ.data(), HW, cudaMemcpyHostToDevice, st));
    env.occ = occb.as<uint8_t>();

    int n_act = 0, cur = 0;
    EP_CUDA(cudaMemcpyAsync(&n_act, cnt.p, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
    EP_CUDA(cudaStreamSynchronize(st));
    if (no == 0) n_act = 0;
    std::vector<int32_t> hmode, haidx;
    for (int step = 0; step < MS && n_act > 0; ++step) {
        k_fill_u32<<<(no + 255) / 256, 256, 0, st>>>(root_step, no, (uint32_t)step);
        for (int off = 0; off < n_act; off += wave) {
            const int nw = std::min(wave, n_act - off);
            const int32_t *act_w = act_list.as<int32_t>() + off;
            RootBatch rb{bel[cur].as<float>(), (long long)m->HWp, (long long)no, root_step, root_ep, act_w, nw};
            m->cur_leaf = QVTS_LEAF_QMDP;
            if (cfg->planner == QVTS_PLANNER_QVTS) {
                qvts_plan_cfg pc{cfg->depth, cfg->n_samples, cfg->seed, 0u, 0u, 0, QVTS_LEAF_QMDP, QVTS_SAMPLER_MARGINAL};
                long long nv[kMaxLevels + 1];
                EP_TRY(plan_levels(*m, rb, pc, nullptr, st, nv));
                k_pick_qvts<<<(nw + 127) / 128, 128, 0, st>>>(ea, act_w, nw, m->ql[0].Q.as<double>(), NA,
                                                              act_ids.as<int32_t>());
            } else {
                EP_TRY(root_marginals(*m, rb, st));
                k_mode<<<nw, 256, 0, st>>>(act_w, bel[cur].as<float>(), m->HWp, HW, mode);
                if (cfg->planner == QVTS_PLANNER_MDP) {
                    k_pick_mdp<<<(nw + 127) / 128, 128, 0, st>>>(ea, act_w, nw, mode, m->d_Q64.as<double>(), NA, HW,
                                                                 act_ids.as<int32_t>());
                } else {   // A* on the belief mode, host-side comparator
                    hmode.resize(nw);
                    haidx.resize(nw);
                    EP_CUDA(cudaMemcpyAsync(hmode.data(), mode, sizeof(int32_t) * nw, cudaMemcpyDeviceToHost, st));
                    EP_CUDA(cudaStreamSynchronize(st));
                    for (int w = 0; w < nw; ++w) {
                        const int k = astar_first_move(*m, hmode[w]);
                        int jj = 0;
                        for (int j = 0; j < NA; ++j) if (m->action_id[j] == k) jj = j;
                        haidx[w] = jj;
                    }
                    EP_CUDA(cudaMemcpyAsync(sel_z, haidx.data(), sizeof(int32_t) * nw, cudaMemcpyHostToDevice, st));
                    k_set_actions<<<(nw + 127) / 128, 128, 0, st>>>(ea, act_w, nw, sel_z, act_ids.as<int32_t>());
                }
            }
            env.P = m->ql[0].P.as<double>();
            k_env<<<(nw + 127) / 128, 128, 0, st>>>(ea, env, act_w, nw);
            EP_CUDA(cudaGetLastError());
            EP_TRY(correct_selected(*m, rb, sel_q, sel_z, sel_out, nw, bel[1 - cur].as<float>(), m->HWp, st));
        }
        // beliefs of finished episodes are no longer read; swap for the survivors
        // (survivors were all written into bel[1-cur] this step)
        cur = 1 - cur;
        k_compact<<<1, 1024, 0, st>>>(ea.outcome, no, act_list.as<int32_t>(), cnt.as<int32_t>());
        EP_CUDA(cudaGetLastError());
        EP_CUDA(cudaMemcpyAsync(&n_act, cnt.p, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
        EP_CUDA(cudaStreamSynchronize(st));
        prof_collect(*m);               // fold this step's instrumentation events (if enabled)
    }
    EP_CUDA(cudaMemsetAsync(recbuf.p, 0, sizeof(double) * 6 * std::max(1, E), st));
    if (no > 0) k_records<<<(no + 127) / 128, 128, 0, st>>>(ea, recbuf.as<double>(), E);
    EP_CUDA(cudaGetLastError());
    if (comm && G > 1) {
        if (comm->allreduce_sum_f64(comm->ctx, recbuf.as<double>(), 6LL * E, (void *)st) != 0) {
            set_error("allreduce callback failed");
            cleanup();
            return QVTS_ERR_COMM;
        }
    }
    std::vector<double> rec((size_t)6 * std::max(1, E));
    EP_CUDA(cudaMemcpyAsync(rec.data(), recbuf.p, sizeof(double) * 6 * std::max(1, E), cudaMemcpyDeviceToHost, st));
    std::vector<int32_t> hl;
    if (want_log) {
        hl.resize((size_t)3 * nn * MS);
        EP_CUDA(cudaMemcpyAsync(hl.data(), logs.p, sizeof(int32_t) * hl.size(), cudaMemcpyDeviceToHost, st));
    }
    EP_CUDA(cudaStreamSynchronize(st));
    for (int e = 0; e < E; ++e) {
        out_host[e].outcome = (int32_t)rec[6 * e];
        out_host[e].steps = (int32_t)rec[6 * e + 1];
        out_host[e].collisions = (int32_t)rec[6 * e + 2];
        out_host[e].x0 = (int32_t)rec[6 * e + 3];
        out_host[e].x_final = (int32_t)rec[6 * e + 4];
        out_host[e].disc_return = rec[6 * e + 5];
    }
    if (want_log)
        for (int i = 0; i < no; ++i) {
            const int e = owned[i];
            for (int t = 0; t < MS; ++t) {
                if (cfg->log_actions) cfg->log_actions[(size_t)e * MS + t] = hl[(size_t)i * MS + t];
                if (cfg->log_obs) cfg->log_obs[(size_t)e * MS + t] = hl[(size_t)nn * MS + (size_t)i * MS + t];
                if (cfg->log_states) cfg->log_states[(size_t)e * MS + t] = hl[(size_t)2 * nn * MS + (size_t)i * MS + t];
            }
        }
    occb.release();
    cleanup();
    return QVTS_OK;
}
