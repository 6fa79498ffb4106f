// bestfirst.cu — the paper's anytime best-first QVTS (Alg. 1 inner loop, Algs. 2-7, Eq. 8;
// PAPER.md:130-298; reading B5).
//
// The tree lives in a device node pool (SoA).  Per iteration the host launches: S1-S3 on the one
// selected V-node (the level kernels, same Philox keys as qvts_plan_step), S4 of its children
// straight into the pool, the Alg. 5 leaf bounds of the new children (fp64 dot products with the
// FIB and PBVI alpha-vectors, chunked over cells with the vectors staged in shared memory), and a
// single-thread Alg. 6/7 backup from the new Q-nodes up to the root, which also publishes root.E
// (findVNodeToExpand) for the next iteration.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstring>
#include <vector>

#include "qvts_internal.cuh"

namespace qvts {

namespace {

struct BfSummary {
    int32_t sel, depth, la0, pad;
    double U, L, H;
};

// VT[x][k]: FIB alpha (k < NA), PBVI alpha (NA <= k < NA + nal), 1 (k = nvec - 1; gives sum b)
__global__ void k_bf_vt(const double *__restrict__ A, int NA, const double *__restrict__ G, int nal, int HW,
                        double *__restrict__ VT) {
    const int nvec = NA + nal + 1;
    const long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (t >= (long long)HW * nvec) return;
    const int x = (int)(t / nvec), k = (int)(t % nvec);
    double v;
    if (k < NA) v = A[(size_t)k * HW + x];
    else if (k < NA + nal) v = G[(size_t)(k - NA) * HW + x];
    else v = 1.0;
    VT[t] = v;
}

// partial dot products of nc beliefs with every vector over one chunk of CH cells
__global__ void __launch_bounds__(256) k_bf_leaf_part(const float *__restrict__ bel, long long stride, int nc,
                                                      const double *__restrict__ VT, int nvec, int HW, int CH,
                                                      double *__restrict__ part) {
    extern __shared__ double vts[];
    const int x0 = blockIdx.x * CH;
    const int cnt = min(CH, HW - x0);
    for (int i = threadIdx.x; i < cnt * nvec; i += 256) vts[i] = VT[(size_t)x0 * nvec + i];
    __syncthreads();
    for (int p = threadIdx.x; p < nc * nvec; p += 256) {
        const int c = p / nvec, k = p % nvec;
        const float *__restrict__ b = bel + (size_t)c * stride + x0;
        double acc = 0.0;
        for (int x = 0; x < cnt; ++x) acc = fma(vts[x * nvec + k], (double)__ldg(b + x), acc);
        part[((size_t)blockIdx.x * nc + c) * nvec + k] = acc;
    }
}

// Alg. 5 for node0 + c: U = max_a alpha_FIB.b / sum b, L = max_k alpha_PBVI.b / sum b (fixed chunk
// order), H = U - L (0 at max_depth), E = self
__global__ void k_bf_leaf_fin(const double *__restrict__ part, int nchunks, int nc, int nvec, int NA, int nal,
                              long long node0, int depth, int max_depth, double *__restrict__ vU,
                              double *__restrict__ vL, double *__restrict__ vH, int32_t *__restrict__ vE,
                              int32_t *__restrict__ vq0, int32_t *__restrict__ vLa, int32_t *__restrict__ vdepth) {
    extern __shared__ double S[];
    const int c = blockIdx.x;
    for (int k = threadIdx.x; k < nvec; k += blockDim.x) {
        double s = 0.0;
        for (int ch = 0; ch < nchunks; ++ch) s += part[((size_t)ch * nc + c) * nvec + k];
        S[k] = s;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        const double s1 = S[nvec - 1];
        double U = 0.0, L = 0.0;
        int la = 0;
        for (int k = 0; k < NA; ++k) {
            const double v = S[k] / s1;
            if (k == 0 || v > U) U = v;
        }
        for (int k = 0; k < nal; ++k) {
            const double v = S[NA + k] / s1;
            if (k == 0 || v > L) { L = v; la = k; }
        }
        const long long i = node0 + c;
        vU[i] = U;
        vL[i] = L;
        vH[i] = depth >= max_depth ? 0.0 : U - L;
        vE[i] = (int32_t)i;
        vq0[i] = -1;
        vLa[i] = la;
        vdepth[i] = depth;
    }
}

__global__ void k_bf_init_root(uint64_t *path, int32_t *pq, int32_t *z, int32_t *f, int32_t *root, int n) {
    path[0] = 0; pq[0] = -1; z[0] = 0; f[0] = n; root[0] = 0;
}

struct BackupArgs {
    int sel, NA, n;
    long long cbase, qbase;
    double gamma;
    const double *R;          // [NA] R(b,a) of the expanded node
    const int32_t *U, *off;   // children per Q-node and offsets
    int32_t *pq, *f, *depth, *vE, *vq0;
    double *vU, *vL, *vH;
    double *qR, *qU, *qL, *qH;
    int32_t *qE, *qc0, *qnc, *qv;
    const int32_t *vLa;
    BfSummary *sum;
};

__device__ void bf_q_update(const BackupArgs &a, long long q) {
    const long long c0 = a.qc0[q];
    const int nc = a.qnc[q];
    double su = 0.0, sl = 0.0, bh = 0.0;
    long long bc = c0;
    for (int i = 0; i < nc; ++i) {
        const long long c = c0 + i;
        const double w = (double)a.f[c] / (double)a.n;
        su += w * a.vU[c];
        sl += w * a.vL[c];
        const double h = a.gamma * w * a.vH[c];                 // Alg. 6: gamma x weight x heuristic
        if (i == 0 || h > bh) { bh = h; bc = c; }
    }
    a.qU[q] = a.qR[q] + a.gamma * su;                           // Alg. 6 with gamma (R13)
    a.qL[q] = a.qR[q] + a.gamma * sl;
    a.qH[q] = bh;
    a.qE[q] = a.vE[bc];
}

__device__ void bf_v_update(const BackupArgs &a, long long v) {
    const long long q0 = a.vq0[v];
    long long bq = q0;
    double bl = a.qL[q0];
    for (int j = 1; j < a.NA; ++j) {
        const long long q = q0 + j;
        if (a.qU[q] > a.qU[bq]) bq = q;                         // H(b,a) = 1 at argmax U_Q (Sec. IV-C)
        if (a.qL[q] > bl) bl = a.qL[q];
    }
    a.vU[v] = a.qU[bq];
    a.vL[v] = bl;
    a.vH[v] = a.qH[bq];
    a.vE[v] = a.qE[bq];
}

__global__ void k_bf_backup(BackupArgs a) {
    const int v = a.sel;
    for (int j = 0; j < a.NA; ++j) {
        const long long q = a.qbase + j;
        a.qR[q] = a.R[j];
        a.qc0[q] = (int32_t)(a.cbase + a.off[j]);
        a.qnc[q] = a.U[j];
        a.qv[q] = v;
        for (int i = 0; i < a.U[j]; ++i) a.pq[a.cbase + a.off[j] + i] = (int32_t)q;
        bf_q_update(a, q);
    }
    a.vq0[v] = (int32_t)a.qbase;
    bf_v_update(a, v);
    for (int p = a.pq[v]; p >= 0;) {                            // p.update() up to the root (Alg. 1)
        bf_q_update(a, p);
        const int pv = a.qv[p];
        bf_v_update(a, pv);
        p = a.pq[pv];
    }
    const int e = a.vE[0];
    a.sum->sel = e;
    a.sum->depth = a.depth[e];
    a.sum->la0 = a.vLa[0];
    a.sum->U = a.vU[0];
    a.sum->L = a.vL[0];
    a.sum->H = a.vH[0];
}

}  // namespace

static qvts_status bf_leaf_bounds(Model &m, long long node0, int nc, int depth, int max_depth, int nvec, int nal,
                                  cudaStream_t st) {
    if (nc == 0) return QVTS_OK;
    const int HW = m.HW;
    int CH = (int)std::min<long long>(512, (150 * 1024) / (8LL * nvec));
    CH = std::max(1, CH >= 32 ? (CH & ~31) : CH);
    const int nchunks = (HW + CH - 1) / CH;
    QVTS_TRY(m.bf_part.ensure(sizeof(double) * (size_t)nchunks * nc * nvec));
    const size_t smem = sizeof(double) * (size_t)CH * nvec;
    QVTS_CUDA(cudaFuncSetAttribute(k_bf_leaf_part, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    k_bf_leaf_part<<<nchunks, 256, smem, st>>>(m.bf_bel.as<float>() + (size_t)node0 * m.HWp, m.HWp, nc,
                                               m.bf_VT.as<double>(), nvec, HW, CH, m.bf_part.as<double>());
    QVTS_CUDA(cudaGetLastError());
    const size_t smem2 = sizeof(double) * nvec;
    QVTS_CUDA(cudaFuncSetAttribute(k_bf_leaf_fin, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem2));
    k_bf_leaf_fin<<<nc, 128, smem2, st>>>(m.bf_part.as<double>(), nchunks, nc, nvec, m.NA, nal, node0, depth,
                                          max_depth, m.bf_vU.as<double>(), m.bf_vL.as<double>(),
                                          m.bf_vH.as<double>(), m.bf_vE.as<int32_t>(), m.bf_vq0.as<int32_t>(),
                                          m.bf_vLa.as<int32_t>(), m.bf_depth.as<int32_t>());
    QVTS_CUDA(cudaGetLastError());
    return QVTS_OK;
}

}  // namespace qvts

using namespace qvts;

extern "C" qvts_status qvts_plan_best_first(qvts_model *m, const float *root_dev, const qvts_bf_cfg *cfg,
                                            qvts_bf_result *res, void *stream) {
    if (!m || !root_dev || !cfg || !res) { set_error("NULL argument"); return QVTS_ERR_INVALID_ARG; }
    if (cfg->n_samples < 1 || cfg->n_samples > 4096 || cfg->max_expansions < 0 || cfg->max_depth < 1 ||
        cfg->max_depth > 8 || !(cfg->gap_tol >= 0.0) ||
        (cfg->sampler != QVTS_SAMPLER_MARGINAL && cfg->sampler != QVTS_SAMPLER_ANCESTRAL)) {
        set_error("bad best-first config (n 1..4096, max_expansions >= 0, max_depth 1..8, gap_tol >= 0)");
        return QVTS_ERR_INVALID_ARG;
    }
    if (!m->have_fib) { set_error("run qvts_fib_iteration before best-first planning"); return QVTS_ERR_STATE; }
    if (!m->have_pbvi) { set_error("run qvts_pbvi before best-first planning"); return QVTS_ERR_STATE; }
    QVTS_CUDA(cudaSetDevice(m->device));
    cudaStream_t st = (cudaStream_t)stream;
    const auto t_start = std::chrono::steady_clock::now();
    const int NA = m->NA, HW = m->HW, n = cfg->n_samples;
    const int nal = m->pb_nal, nvec = NA + nal + 1;
    // node pool capacity
    const long long per_exp = (long long)NA * std::min(n, 16);
    long long cap_v = 1 + (long long)cfg->max_expansions * per_exp;
    size_t free_b = 0, total_b = 0;
    QVTS_CUDA(cudaMemGetInfo(&free_b, &total_b));
    const long long by_mem = std::max(1LL, (long long)(free_b / 2 / ((size_t)m->HWp * 4 + 128)));
    cap_v = std::max(1LL, std::min(cap_v, by_mem));
    const long long cap_q = std::max(1LL, (long long)cfg->max_expansions * NA);
    m->bf_valid = false;
    QVTS_TRY(m->bf_bel.ensure(sizeof(float) * (size_t)cap_v * m->HWp));
    QVTS_TRY(m->bf_path.ensure(sizeof(uint64_t) * cap_v));
    for (DevBuf *b : {&m->bf_pq, &m->bf_z, &m->bf_f, &m->bf_root, &m->bf_depth, &m->bf_vE, &m->bf_vq0, &m->bf_vLa})
        QVTS_TRY(b->ensure(sizeof(int32_t) * cap_v));
    for (DevBuf *b : {&m->bf_vU, &m->bf_vL, &m->bf_vH}) QVTS_TRY(b->ensure(sizeof(double) * cap_v));
    for (DevBuf *b : {&m->bf_qR, &m->bf_qU, &m->bf_qL, &m->bf_qH}) QVTS_TRY(b->ensure(sizeof(double) * cap_q));
    for (DevBuf *b : {&m->bf_qE, &m->bf_qc0, &m->bf_qnc, &m->bf_qv}) QVTS_TRY(b->ensure(sizeof(int32_t) * cap_q));
    QVTS_TRY(m->bf_VT.ensure(sizeof(double) * (size_t)HW * nvec));
    QVTS_TRY(m->bf_sum.ensure(sizeof(BfSummary)));
    QVTS_TRY(m->bf_keys.ensure(sizeof(uint32_t) * 2));
    uint32_t keys[2] = {cfg->step, cfg->episode};
    QVTS_CUDA(cudaMemcpyAsync(m->bf_keys.p, keys, sizeof(keys), cudaMemcpyHostToDevice, st));
    const uint32_t *kstep = m->bf_keys.as<uint32_t>(), *kep = kstep + 1;

    QVTS_CUDA(cudaEventRecord(m->ev0, st));
    k_bf_vt<<<(unsigned)(((long long)HW * nvec + 255) / 256), 256, 0, st>>>(m->d_alpha64.as<double>(), NA,
                                                                              m->pb_G.as<double>(), nal, HW,
                                                                              m->bf_VT.as<double>());
    QVTS_CUDA(cudaMemcpyAsync(m->bf_bel.p, root_dev, sizeof(float) * HW, cudaMemcpyDeviceToDevice, st));
    k_bf_init_root<<<1, 1, 0, st>>>(m->bf_path.as<uint64_t>(), m->bf_pq.as<int32_t>(), m->bf_z.as<int32_t>(),
                                    m->bf_f.as<int32_t>(), m->bf_root.as<int32_t>(), n);
    QVTS_CUDA(cudaGetLastError());
    QVTS_TRY(bf_leaf_bounds(*m, 0, 1, 0, cfg->max_depth, nvec, nal, st));
    // the root summary straight from its leaf values
    BfSummary sum{};
    {
        double u[3];
        int32_t la = 0;
        QVTS_CUDA(cudaMemcpyAsync(&u[0], m->bf_vU.p, sizeof(double), cudaMemcpyDeviceToHost, st));
        QVTS_CUDA(cudaMemcpyAsync(&u[1], m->bf_vL.p, sizeof(double), cudaMemcpyDeviceToHost, st));
        QVTS_CUDA(cudaMemcpyAsync(&u[2], m->bf_vH.p, sizeof(double), cudaMemcpyDeviceToHost, st));
        QVTS_CUDA(cudaMemcpyAsync(&la, m->bf_vLa.p, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
        QVTS_CUDA(cudaStreamSynchronize(st));
        sum.sel = 0; sum.depth = 0; sum.la0 = la; sum.U = u[0]; sum.L = u[1]; sum.H = u[2];
    }
    long long nv = 1, nq = 0;
    int nexp = 0, stop = QVTS_BF_BUDGET;
    m->bf_exp.clear();
    m->bf_rtrace.clear();
    for (;;) {
        m->bf_rtrace.push_back(sum.U);
        m->bf_rtrace.push_back(sum.L);
        if (nexp >= cfg->max_expansions) { stop = QVTS_BF_BUDGET; break; }
        if (sum.U - sum.L <= cfg->gap_tol) { stop = QVTS_BF_GAP; break; }
        if (sum.depth >= cfg->max_depth) { stop = QVTS_BF_TERMINAL; break; }
        if (nv + per_exp > cap_v) { stop = QVTS_BF_POOL; break; }
        if (cfg->time_budget_ms > 0.0 &&
            std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t_start).count() >=
                cfg->time_budget_ms) {
            stop = QVTS_BF_TIME;
            break;
        }
        const int v = sum.sel;
        ExpandSpec e;
        e.beliefs = m->bf_bel.as<float>() + (size_t)v * m->HWp;
        e.bstride = m->HWp; e.nwork = 1;
        e.vpath = m->bf_path.as<uint64_t>() + v;
        e.vroot = m->bf_root.as<int32_t>() + v;
        e.root_step = kstep; e.root_ep = kep;
        e.level = sum.depth; e.n = n; e.seed = cfg->seed; e.sampler = cfg->sampler;
        long long total = 0;
        QVTS_TRY(expand_marginals(*m, e, m->bf_ql, st, &total));
        ChildOut o;
        o.belief = m->bf_bel.as<float>() + (size_t)nv * m->HWp;
        o.stride = m->HWp;
        o.path = m->bf_path.as<uint64_t>() + nv;
        o.parent_q = m->bf_pq.as<int32_t>() + nv;
        o.z = m->bf_z.as<int32_t>() + nv;
        o.f = m->bf_f.as<int32_t>() + nv;
        o.root = m->bf_root.as<int32_t>() + nv;
        QVTS_TRY(expand_children(*m, e, m->bf_ql, o, st));
        QVTS_TRY(bf_leaf_bounds(*m, nv, (int)total, sum.depth + 1, cfg->max_depth, nvec, nal, st));
        BackupArgs a;
        a.sel = v; a.NA = NA; a.n = n; a.cbase = nv; a.qbase = nq; a.gamma = m->gamma;
        a.R = m->bf_ql.R.as<double>(); a.U = m->bf_ql.U.as<int32_t>(); a.off = m->bf_ql.off.as<int32_t>();
        a.pq = m->bf_pq.as<int32_t>(); a.f = m->bf_f.as<int32_t>(); a.depth = m->bf_depth.as<int32_t>();
        a.vE = m->bf_vE.as<int32_t>(); a.vq0 = m->bf_vq0.as<int32_t>();
        a.vU = m->bf_vU.as<double>(); a.vL = m->bf_vL.as<double>(); a.vH = m->bf_vH.as<double>();
        a.qR = m->bf_qR.as<double>(); a.qU = m->bf_qU.as<double>(); a.qL = m->bf_qL.as<double>();
        a.qH = m->bf_qH.as<double>(); a.qE = m->bf_qE.as<int32_t>(); a.qc0 = m->bf_qc0.as<int32_t>();
        a.qnc = m->bf_qnc.as<int32_t>(); a.qv = m->bf_qv.as<int32_t>(); a.vLa = m->bf_vLa.as<int32_t>();
        a.sum = m->bf_sum.as<BfSummary>();
        k_bf_backup<<<1, 1, 0, st>>>(a);
        QVTS_CUDA(cudaGetLastError());
        QVTS_CUDA(cudaMemcpyAsync(&sum, m->bf_sum.p, sizeof(BfSummary), cudaMemcpyDeviceToHost, st));
        QVTS_CUDA(cudaStreamSynchronize(st));
        m->bf_exp.push_back(v);
        nv += total;
        nq += NA;
        ++nexp;
    }
    QVTS_CUDA(cudaEventRecord(m->ev1, st));
    std::memset(res, 0, sizeof(*res));
    res->n_actions = NA;
    res->n_expansions = nexp;
    res->stop_reason = stop;
    res->n_vnodes = nv;
    res->U = sum.U;
    res->L = sum.L;
    for (int j = 0; j < 9; ++j) res->u_q[j] = res->l_q[j] = NAN;
    if (nexp > 0) {   // the root was expanded first: its Q-nodes are 0..NA-1
        QVTS_CUDA(cudaMemcpyAsync(res->u_q, m->bf_qU.p, sizeof(double) * NA, cudaMemcpyDeviceToHost, st));
        QVTS_CUDA(cudaMemcpyAsync(res->l_q, m->bf_qL.p, sizeof(double) * NA, cudaMemcpyDeviceToHost, st));
    }
    QVTS_CUDA(cudaStreamSynchronize(st));
    float ms = 0.f;
    QVTS_CUDA(cudaEventElapsedTime(&ms, m->ev0, m->ev1));
    res->device_ms = ms;
    if (nexp == 0) {
        res->action = m->pb_act[sum.la0];
    } else {                  // getOptimalAction: max L_Q, ties by U_Q then index
        int best = 0;
        for (int j = 1; j < NA; ++j)
            if (res->l_q[j] > res->l_q[best] || (res->l_q[j] == res->l_q[best] && res->u_q[j] > res->u_q[best])) best = j;
        res->action = m->action_id[best];
    }
    m->bf_nv = nv;
    m->bf_nq = nq;
    m->bf_nexp = nexp;
    m->bf_valid = true;
    prof_collect(*m);
    return QVTS_OK;
}

extern "C" qvts_status qvts_trace_best_first(const qvts_model *m, int64_t *n_v, int32_t *n_expansions, uint64_t *path,
                                             int32_t *depth, int32_t *f, double *U, double *L, double *H, int32_t *E,
                                             int32_t *expanded, int32_t *exp_order, double *root_trace) {
    if (!m) { set_error("model is NULL"); return QVTS_ERR_INVALID_ARG; }
    if (!m->bf_valid) { set_error("qvts_plan_best_first has not run"); return QVTS_ERR_STATE; }
    QVTS_CUDA(cudaSetDevice(m->device));
    const size_t nv = (size_t)m->bf_nv;
    if (n_v) *n_v = m->bf_nv;
    if (n_expansions) *n_expansions = m->bf_nexp;
    if (path) QVTS_CUDA(cudaMemcpy(path, m->bf_path.p, sizeof(uint64_t) * nv, cudaMemcpyDeviceToHost));
    if (depth) QVTS_CUDA(cudaMemcpy(depth, m->bf_depth.p, sizeof(int32_t) * nv, cudaMemcpyDeviceToHost));
    if (f) QVTS_CUDA(cudaMemcpy(f, m->bf_f.p, sizeof(int32_t) * nv, cudaMemcpyDeviceToHost));
    if (U) QVTS_CUDA(cudaMemcpy(U, m->bf_vU.p, sizeof(double) * nv, cudaMemcpyDeviceToHost));
    if (L) QVTS_CUDA(cudaMemcpy(L, m->bf_vL.p, sizeof(double) * nv, cudaMemcpyDeviceToHost));
    if (H) QVTS_CUDA(cudaMemcpy(H, m->bf_vH.p, sizeof(double) * nv, cudaMemcpyDeviceToHost));
    if (E) QVTS_CUDA(cudaMemcpy(E, m->bf_vE.p, sizeof(int32_t) * nv, cudaMemcpyDeviceToHost));
    if (expanded) {
        std::vector<int32_t> q0(nv);
        QVTS_CUDA(cudaMemcpy(q0.data(), m->bf_vq0.p, sizeof(int32_t) * nv, cudaMemcpyDeviceToHost));
        for (size_t i = 0; i < nv; ++i) expanded[i] = q0[i] >= 0 ? 1 : 0;
    }
    if (exp_order) std::memcpy(exp_order, m->bf_exp.data(), sizeof(int32_t) * m->bf_exp.size());
    if (root_trace) std::memcpy(root_trace, m->bf_rtrace.data(), sizeof(double) * m->bf_rtrace.size());
    return QVTS_OK;
}
