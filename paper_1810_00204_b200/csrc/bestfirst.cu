// bestfirst.cu — the paper's anytime best-first QVTS (Alg. 1 inner loop, Algs. 2-7, Eq. 8;
// PAPER.md:130-298; reading B5).
//
// The tree lives in a device node pool (SoA) and the loop state (root.E, pool fill, stop flag) in
// device memory, so one expansion is a fixed launch sequence that a CUDA graph replays: S1-S3 on
// the selected V-node (the level kernels, same Philox keys as qvts_plan_step), S4 of its children
// straight into the pool, the Alg. 5 leaf bounds of the new children (fp64 split-K dot products
// with the FIB and PBVI alpha-vectors), and a one-CTA Alg. 6/7 backup from the new Q-nodes up to
// the root, which publishes root.E (findVNodeToExpand) and evaluates planningFinished().  The host
// replays the graph in chunks and reads the state back between chunks (time budget, pool growth).
#include <algorithm>
#include <chrono>
#include <climits>
#include <cmath>
#include <cstring>
#include <vector>

#include "qvts_internal.cuh"

namespace qvts {

// bracket one launch with instrumentation events (no-op unless profiling is on)
#define QVTS_BF_PROF(model, cat, ...)             \
    do {                                          \
        cudaEvent_t e__;                          \
        prof_begin(model, cat, st, &e__);         \
        __VA_ARGS__;                              \
        prof_end(model, cat, st, e__);            \
    } while (0)

namespace {

// loop state in device memory
struct BfDev {
    int32_t sel, depth;           // root.E and its depth (depth = -1 while the root is built)
    int32_t done, stop;           // planningFinished() and its qvts_bf_stop reason
    int32_t nexp, la0;            // expansions done; PBVI arg-max vector of the root
    long long nv, nq;             // pool fill (V-nodes, Q-nodes)
    long long total;              // children of the current expansion
    long long cap_v;              // pool capacity (V-nodes)
    double U, L, H;               // root bounds and heuristic
    int32_t budget, max_depth, per_exp, root;   // root: pool index of the current root
    double gap_tol;
};

// planningFinished() after the state has been updated (Alg. 1, reading B5)
__device__ void bf_check_done(BfDev *S) {
    int stop = -1;
    if (S->nexp >= S->budget) stop = QVTS_BF_BUDGET;
    else if (S->U - S->L <= S->gap_tol) stop = QVTS_BF_GAP;
    else if (S->depth >= S->max_depth) stop = QVTS_BF_TERMINAL;
    else if (S->nv + S->per_exp > S->cap_v) stop = QVTS_BF_POOL;
    if (stop >= 0) { S->done = 1; S->stop = stop; }
}

// VK[k][x]: FIB alpha (k < NA), PBVI alpha (NA <= k < NA + nal), 1 (k = nvec - 1: gives sum b),
// zero rows up to the padded vector count
__global__ void k_bf_vk(const double *__restrict__ A, int NA, const double *__restrict__ G, int nal, int HW,
                        int nrows, double *__restrict__ VK) {
    const long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (t >= (long long)HW * nrows) return;
    const int k = (int)(t / HW), x = (int)(t % HW);
    double v = 0.0;
    if (k < NA) v = A[(size_t)k * HW + x];
    else if (k < NA + nal) v = G[(size_t)(k - NA) * HW + x];
    else if (k == NA + nal) v = 1.0;
    VK[t] = v;
}

// S[c][k] = sum_x b_c(x) VK[k][x] as a split-K product: CTA (s, kb) takes cells [s XS, (s+1) XS)
// and vectors [kb 16 KJ, +16 KJ).  The whole slice of beliefs (fp32) and vectors (fp64) is staged
// into shared memory with one burst of cp.async (row pitch XS + 1: the 16 rows a warp reads sit in
// distinct banks), then thread (tc, tk) accumulates a CI x KJ register tile of
// (c = tc + 16 i, k = tk + 16 j) in fp64.
template <int CI, int KJ>
__global__ void __launch_bounds__(256) k_bf_dots(const float *__restrict__ bel_pool, long long stride,
                                                 const BfDev *__restrict__ S, const double *__restrict__ VK, int HW,
                                                 int XS, int nsplit, double *__restrict__ part) {
    extern __shared__ double smd[];
    if (S->done) return;
    // children of this expansion: pool slots [nv, nv + total) (the root alone when depth < 0)
    const long long node0 = S->depth < 0 ? 0 : S->nv;
    const int nc_all = S->depth < 0 ? 1 : (int)S->total;
    const int cg = blockIdx.z * 16 * CI;                               // this CTA's first child
    if (cg >= nc_all) return;
    const int nc = min(16 * CI, nc_all - cg);
    const float *__restrict__ bel = bel_pool + (size_t)(node0 + cg) * stride;
    const int P = XS + 1;
    double *Vs = smd;                                                // [16 KJ][P]
    float *Bs = reinterpret_cast<float *>(smd + 16 * KJ * P);         // [16 CI][P]
    const int tid = threadIdx.x, tc = tid >> 4, tk = tid & 15;
    const int kbase = blockIdx.y * 16 * KJ;
    const int x0 = blockIdx.x * XS, n = min(XS, HW - x0);
    for (int i = tid; i < 16 * KJ * XS; i += 256) {
        const int k = i / XS, xx = i % XS;
        const bool ok = xx < n;
        const double *src = VK + (size_t)(kbase + k) * HW + x0 + (ok ? xx : 0);
        const unsigned dst = (unsigned)__cvta_generic_to_shared(Vs + k * P + xx);
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(dst), "l"(src), "r"(ok ? 8 : 0));
    }
    for (int i = tid; i < 16 * CI * XS; i += 256) {
        const int c = i / XS, xx = i % XS;
        const bool ok = xx < n && c < nc;
        const float *src = bel + (ok ? (size_t)c * stride + x0 + xx : 0);
        const unsigned dst = (unsigned)__cvta_generic_to_shared(Bs + c * P + xx);
        asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;\n" ::"r"(dst), "l"(src), "r"(ok ? 4 : 0));
    }
    asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;\n" ::: "memory");
    __syncthreads();
    double acc[CI][KJ];
#pragma unroll
    for (int i = 0; i < CI; ++i)
#pragma unroll
        for (int j = 0; j < KJ; ++j) acc[i][j] = 0.0;
#pragma unroll 4
    for (int xx = 0; xx < n; ++xx) {
        double b[CI], v[KJ];
#pragma unroll
        for (int i = 0; i < CI; ++i) b[i] = (double)Bs[(tc + 16 * i) * P + xx];
#pragma unroll
        for (int j = 0; j < KJ; ++j) v[j] = Vs[(tk + 16 * j) * P + xx];
#pragma unroll
        for (int i = 0; i < CI; ++i)
#pragma unroll
            for (int j = 0; j < KJ; ++j) acc[i][j] = fma(b[i], v[j], acc[i][j]);
    }
    // part [kb][split][child 0..143][16 KJ]
    double *out = part + (((size_t)blockIdx.y * nsplit + blockIdx.x) * 144 + cg) * (16 * KJ);
#pragma unroll
    for (int i = 0; i < CI; ++i)
#pragma unroll
        for (int j = 0; j < KJ; ++j) out[(tc + 16 * i) * (16 * KJ) + tk + 16 * j] = acc[i][j];
}

// Alg. 5 for node0 + c: U = max_a alpha_FIB.b / sum b, L = max_k alpha_PBVI.b / sum b, H = U - L
// (0 at max_depth: terminal), E = self.  Block (32, 32): lane x = vector k mod 32, row y sums the
// splits sp = y, y + 32, ... in ascending order; the 32 row sums are added in row order.
__global__ void __launch_bounds__(1024) k_bf_leaf_fin(const double *__restrict__ part, int nsplit, int KB,
                                                      int nvec, int NA, int nal, const BfDev *__restrict__ St,
                                                      double *__restrict__ vU, double *__restrict__ vL,
                                                      double *__restrict__ vH, int32_t *__restrict__ vE,
                                                      int32_t *__restrict__ vq0, int32_t *__restrict__ vLa,
                                                      int32_t *__restrict__ vdepth) {
    extern __shared__ double S[];          // [nvec]
    __shared__ double rows[32][33];
    const int c = blockIdx.x, tx = threadIdx.x, ty = threadIdx.y;
    if (St->done) return;
    const bool root = St->depth < 0;
    if (c >= (root ? 1 : (int)St->total)) return;
    const long long node0 = root ? 0 : St->nv;
    const int depth = St->depth + 1, max_depth = St->max_depth;
    const int CIP = 144;
    for (int k0 = 0; k0 < nvec; k0 += 32) {
        const int k = k0 + tx;
        double s = 0.0;
        if (k < nvec) {
            const int kb = k / KB, kk = k % KB;
            for (int sp = ty; sp < nsplit; sp += 32) s += part[(((size_t)kb * nsplit + sp) * CIP + c) * KB + kk];
        }
        rows[ty][tx] = s;
        __syncthreads();
        if (ty == 0 && k < nvec) {
            double t = 0.0;
            for (int r = 0; r < 32; ++r) t += rows[r][tx];
            S[k] = t;
        }
        __syncthreads();
    }
    if (tx == 0 && ty == 0) {
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

// after the root's leaf bounds: s = QVSearchTree(b0) (Alg. 1), root.E = root
__global__ void k_bf_root_state(BfDev *S, const double *vU, const double *vL, const double *vH, const int32_t *vLa,
                                double *rtrace) {
    S->root = 0; S->sel = 0; S->depth = 0; S->nv = 1; S->nq = 0; S->nexp = 0; S->total = 0;
    S->U = vU[0]; S->L = vL[0]; S->H = vH[0]; S->la0 = vLa[0];
    rtrace[0] = S->U;
    rtrace[1] = S->L;
    bf_check_done(S);
}

// tree reuse (NEXT-4): resume from the kept tree's root -- root.E, bounds, a fresh per-call count
__global__ void k_bf_resume(BfDev *S, const int32_t *vE, const int32_t *vdepth, const double *vU, const double *vL,
                            const double *vH, const int32_t *vLa, double *rtrace) {
    const int r = S->root;
    S->sel = vE[r]; S->depth = vdepth[S->sel]; S->nexp = 0; S->total = 0; S->done = 0; S->stop = 0;
    S->U = vU[r]; S->L = vL[r]; S->H = vH[r]; S->la0 = vLa[r];
    rtrace[0] = S->U;
    rtrace[1] = S->L;
    bf_check_done(S);
}

// s.update(a, z) (Alg. 1): re-root at pool node c.  Nodes of its subtree (depth-1 ancestor = c) lose
// one level (path >> 8, depth - 1, ancestor lists shifted); every other node is discarded (depth -1).
__global__ void k_bf_rebase(long long nv, int c, uint64_t *path, int32_t *vdepth, int32_t *anc, int32_t *pq) {
    const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (i >= nv) return;
    const int d = vdepth[i];
    int32_t *an = anc + (size_t)i * 16;
    const bool member = d == 1 ? (i == c) : (d >= 2 && an[1] == c);
    if (!member) { vdepth[i] = -1; return; }
    path[i] >>= 8;
    vdepth[i] = d - 1;
    for (int l = 0; l < 7; ++l) { an[l] = an[l + 1]; an[8 + l] = an[9 + l]; }
    if (i == c) pq[i] = -1;
}

struct BackupArgs {
    BfDev *S;
    int NA, n;
    double gamma;
    const double *R;          // [NA] R(b,a) of the expanded node
    const int32_t *U, *off;   // children per Q-node and offsets
    int32_t *pq, *f, *vdepth, *vE, *vq0, *anc;   // anc: [node][16] = V ancestors by depth, Q ancestors by depth
    double *vU, *vL, *vH;
    double *qR, *qU, *qL, *qH;
    int32_t *qE, *qc0, *qnc, *qv;
    const int32_t *vLa;
    double *rtrace;           // root (U, L) after each expansion
};

// Alg. 6 fold of up to 16 children (ascending, the oracle's order) -> (U_Q, L_Q, H_Q, E_Q)
__device__ __forceinline__ void bf_fold_q(double R, double gamma, int nc, const double *w, const double *U,
                                          const double *L, const double *H, const int *E, double *out4, int *eq) {
    double su = 0.0, sl = 0.0, bh = 0.0;
    int be = 0;
    for (int i = 0; i < nc; ++i) {
        su += w[i] * U[i];
        sl += w[i] * L[i];
        const double h = gamma * w[i] * H[i];                  // Alg. 6: gamma x weight x heuristic
        if (i == 0 || h > bh) { bh = h; be = E[i]; }
    }
    out4[0] = R + gamma * su;                                  // Alg. 6 with gamma (R13)
    out4[1] = R + gamma * sl;
    out4[2] = bh;
    *eq = be;
}

// Alg. 7 fold over the NA Q-children: U = max U_Q, L = max L_Q, (H, E) of the argmax-U child
__device__ __forceinline__ void bf_fold_v(int NA, const double *U, const double *L, const double *H, const int *E,
                                          double *out3, int *ev) {
    int bq = 0;
    double bl = L[0];
    for (int j = 1; j < NA; ++j) {
        if (U[j] > U[bq]) bq = j;                              // H(b,a) = 1 at argmax U_Q (Sec. IV-C)
        if (L[j] > bl) bl = L[j];
    }
    out3[0] = U[bq];
    out3[1] = bl;
    out3[2] = H[bq];
    *ev = E[bq];
}

// One CTA: gather every value the update needs (the new Q-nodes' children, and for each ancestor
// level the Q-node's children and the V-node's Q-children) in one parallel round, recompute
// bottom-up in shared memory (Alg. 6 / Alg. 7 up to the root, Alg. 1), scatter the results.
__global__ void __launch_bounds__(256) k_bf_backup(BackupArgs a) {
    __shared__ int s_ancv[8], s_ancq[8];
    // new Q-nodes: [j][i] children values
    __shared__ double nw[9][16], nU[9][16], nL[9][16], nH[9][16];
    __shared__ int nE[9][16];
    // ancestor levels: Q-node children [l][i], V-node Q-children [l][j]
    __shared__ double aw[8][16], aU[8][16], aL[8][16], aH[8][16];
    __shared__ int aE[8][16], aC[8][16], anc_n[8], aq0[8];
    __shared__ double aR[8];
    __shared__ double bU[8][9], bL[8][9], bH[8][9];
    __shared__ int bE[8][9];
    __shared__ double qv4[9][3];
    __shared__ int qve[9];
    BfDev *S = a.S;
    if (S->done) return;
    const int t = threadIdx.x, NA = a.NA, d = S->depth, v = S->sel;
    const long long cbase = S->nv, qbase = S->nq;
    if (t < d) {
        s_ancv[t] = a.anc[(size_t)v * 16 + t];
        s_ancq[t] = a.anc[(size_t)v * 16 + 8 + t];
    }
    __syncthreads();
    // gather (one parallel round of independent loads)
    if (t < NA * 16) {
        const int j = t >> 4, i = t & 15;
        if (i < a.U[j]) {
            const long long c = cbase + a.off[j] + i;
            nw[j][i] = (double)a.f[c] / (double)a.n;
            nU[j][i] = a.vU[c]; nL[j][i] = a.vL[c]; nH[j][i] = a.vH[c]; nE[j][i] = a.vE[c];
        }
    }
    if (t < d * 16) {
        const int l = t >> 4, i = t & 15;
        const int q = s_ancq[l];
        const int nc = a.qnc[q], c0 = a.qc0[q];
        if (i == 0) { anc_n[l] = nc; aR[l] = a.qR[q]; }
        if (i < nc) {
            const int c = c0 + i;
            aw[l][i] = (double)a.f[c] / (double)a.n;
            aU[l][i] = a.vU[c]; aL[l][i] = a.vL[c]; aH[l][i] = a.vH[c]; aE[l][i] = a.vE[c]; aC[l][i] = c;
        }
    } else if (t >= 128 && t < 128 + d * 16) {
        const int l = (t - 128) >> 4, j = (t - 128) & 15;
        if (j < NA) {
            const int q0 = a.vq0[s_ancv[l]];
            if (j == 0) aq0[l] = q0;
            bU[l][j] = a.qU[q0 + j]; bL[l][j] = a.qL[q0 + j]; bH[l][j] = a.qH[q0 + j]; bE[l][j] = a.qE[q0 + j];
        }
    }
    __syncthreads();
    // the new Q-nodes in parallel (thread j)
    if (t < NA) {
        bf_fold_q(a.R[t], a.gamma, a.U[t], nw[t], nU[t], nL[t], nH[t], nE[t], qv4[t], &qve[t]);
    }
    __syncthreads();
    if (t == 0) {
        double cu[9], cl[9], ch[9], v3[3];
        int ce[9], ev;
        for (int j = 0; j < NA; ++j) { cu[j] = qv4[j][0]; cl[j] = qv4[j][1]; ch[j] = qv4[j][2]; ce[j] = qve[j]; }
        bf_fold_v(NA, cu, cl, ch, ce, v3, &ev);
        a.vU[v] = v3[0]; a.vL[v] = v3[1]; a.vH[v] = v3[2]; a.vE[v] = ev; a.vq0[v] = (int32_t)qbase;
        // up the path: the updated node replaces its old values in its parent's fold
        int child = v;
        double cv[3] = {v3[0], v3[1], v3[2]};
        int cev = ev;
        for (int l = d - 1; l >= 0; --l) {
            const int nc = anc_n[l];
            for (int i = 0; i < nc; ++i)
                if (aC[l][i] == child) { aU[l][i] = cv[0]; aL[l][i] = cv[1]; aH[l][i] = cv[2]; aE[l][i] = cev; }
            double q4[3];
            int qe;
            bf_fold_q(aR[l], a.gamma, nc, aw[l], aU[l], aL[l], aH[l], aE[l], q4, &qe);
            const int q = s_ancq[l];
            a.qU[q] = q4[0]; a.qL[q] = q4[1]; a.qH[q] = q4[2]; a.qE[q] = qe;
            const int jq = q - aq0[l];
            bU[l][jq] = q4[0]; bL[l][jq] = q4[1]; bH[l][jq] = q4[2]; bE[l][jq] = qe;
            bf_fold_v(NA, bU[l], bL[l], bH[l], bE[l], cv, &cev);
            child = s_ancv[l];
            a.vU[child] = cv[0]; a.vL[child] = cv[1]; a.vH[child] = cv[2]; a.vE[child] = cev;
        }
    }
    __syncthreads();   // every thread has read the state before it advances
    // scatter the new Q-nodes and the children's parent / ancestor lists
    if (t < NA) {
        const long long q = qbase + t;
        a.qR[q] = a.R[t];
        a.qc0[q] = (int32_t)(cbase + a.off[t]);
        a.qnc[q] = a.U[t];
        a.qv[q] = v;
        a.qU[q] = qv4[t][0]; a.qL[q] = qv4[t][1]; a.qH[q] = qv4[t][2]; a.qE[q] = qve[t];
    }
    if (t < NA * 16) {
        const int j = t >> 4, i = t & 15;
        if (i < a.U[j]) {
            const long long c = cbase + a.off[j] + i;
            a.pq[c] = (int32_t)(qbase + j);
            int32_t *an = a.anc + (size_t)c * 16;
            for (int l = 0; l < d; ++l) { an[l] = s_ancv[l]; an[8 + l] = s_ancq[l]; }
            an[d] = v;
            an[8 + d] = (int32_t)(qbase + j);
        }
    }
    if (t == 0) {   // publish root.E and the root bounds, advance the pool, planningFinished()
        const int r = S->root;
        const int e = a.vE[r];
        S->sel = e;
        S->depth = a.vdepth[e];
        S->U = a.vU[r];
        S->L = a.vL[r];
        S->H = a.vH[r];
        S->nv = cbase + S->total;
        S->nq = qbase + NA;
        S->nexp += 1;
        a.rtrace[2 * S->nexp] = S->U;
        a.rtrace[2 * S->nexp + 1] = S->L;
        bf_check_done(S);
    }
}

}  // namespace

static int bf_kj(int nvec) { return nvec <= 16 ? 1 : nvec <= 32 ? 2 : 4; }

// geometry of the leaf-bound product for the current alpha sets
struct BfGeom {
    int nvec, nal, KJ, KB, nkb, XS, nsplit;
};

static BfGeom bf_geom(const Model &m) {
    BfGeom g;
    g.nal = m.pb_nal;
    g.nvec = m.NA + g.nal + 1;
    g.KJ = bf_kj(g.nvec);
    g.KB = 16 * g.KJ;
    g.nkb = (g.nvec + g.KB - 1) / g.KB;
    // slice: about two CTAs per SM, the staged slice within 200 KB of shared memory (CI = 3)
    int XS = (m.HW + 2 * 148 - 1) / (2 * 148);
    XS = std::max(32, (XS + 31) & ~31);
    const int xs_cap = std::max(32, ((200 * 1024) / (16 * g.KJ * 8 + 48 * 4) - 1) & ~31);
    g.XS = std::min(XS, xs_cap);
    g.nsplit = (m.HW + g.XS - 1) / g.XS;
    return g;
}

template <int KJ>
static void bf_dots_launch(Model &m, const BfGeom &g, BfDev *S, cudaStream_t st) {
    const size_t smem = (size_t)(g.XS + 1) * (16 * KJ * 8 + 48 * 4);
    // per call (the attribute is per device; the call is cheap and legal during graph capture)
    cudaFuncSetAttribute(k_bf_dots<3, KJ>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    k_bf_dots<3, KJ><<<dim3(g.nsplit, g.nkb, 3), 256, smem, st>>>(m.bf_bel.as<float>(), m.HWp, S, m.bf_VT.as<double>(),
                                                                  m.HW, g.XS, g.nsplit, m.bf_part.as<double>());
}

// Alg. 5 leaf bounds of the new children (or of the root while S->depth < 0)
static qvts_status bf_leaf_bounds(Model &m, const BfGeom &g, BfDev *S, cudaStream_t st) {
    QVTS_BF_PROF(m, 2, {
        if (g.KJ == 1) bf_dots_launch<1>(m, g, S, st);
        else if (g.KJ == 2) bf_dots_launch<2>(m, g, S, st);
        else bf_dots_launch<4>(m, g, S, st);
    });
    QVTS_CUDA(cudaGetLastError());
    QVTS_BF_PROF(m, 7, k_bf_leaf_fin<<<144, dim3(32, 32), sizeof(double) * g.nvec, st>>>(
                           m.bf_part.as<double>(), g.nsplit, g.KB, g.nvec, m.NA, g.nal, S, m.bf_vU.as<double>(),
                           m.bf_vL.as<double>(), m.bf_vH.as<double>(), m.bf_vE.as<int32_t>(), m.bf_vq0.as<int32_t>(),
                           m.bf_vLa.as<int32_t>(), m.bf_depth.as<int32_t>()));
    QVTS_CUDA(cudaGetLastError());
    return QVTS_OK;
}

// one whole expansion (graph body): level kernels on root.E, leaf bounds, backup
static qvts_status bf_one_expansion(Model &m, const BfGeom &g, BfDev *S, const qvts_bf_cfg &cfg, cudaStream_t st) {
    BfLaunch L;
    L.bel = m.bf_bel.as<float>(); L.stride = m.HWp;
    L.path = m.bf_path.as<uint64_t>(); L.pq = m.bf_pq.as<int32_t>(); L.z = m.bf_z.as<int32_t>();
    L.f = m.bf_f.as<int32_t>(); L.root = m.bf_root.as<int32_t>();
    L.sel = &S->sel; L.skip = &S->done; L.cbase = &S->nv; L.total = &S->total;
    L.root_step = m.bf_keys.as<uint32_t>(); L.root_ep = L.root_step + 1;
    L.n = cfg.n_samples; L.seed = cfg.seed; L.sampler = cfg.sampler;
    QVTS_TRY(bf_expand_launch(m, L, m.bf_ql, st));
    QVTS_TRY(bf_leaf_bounds(m, g, S, st));
    BackupArgs a;
    a.S = S; a.NA = m.NA; a.n = cfg.n_samples; a.gamma = m.gamma;
    a.R = m.bf_ql.R.as<double>(); a.U = m.bf_ql.U.as<int32_t>(); a.off = m.bf_ql.off.as<int32_t>();
    a.pq = m.bf_pq.as<int32_t>(); a.f = m.bf_f.as<int32_t>(); a.vdepth = m.bf_depth.as<int32_t>();
    a.anc = m.bf_anc.as<int32_t>();
    a.vE = m.bf_vE.as<int32_t>(); a.vq0 = m.bf_vq0.as<int32_t>();
    a.vU = m.bf_vU.as<double>(); a.vL = m.bf_vL.as<double>(); a.vH = m.bf_vH.as<double>();
    a.qR = m.bf_qR.as<double>(); a.qU = m.bf_qU.as<double>(); a.qL = m.bf_qL.as<double>();
    a.qH = m.bf_qH.as<double>(); a.qE = m.bf_qE.as<int32_t>(); a.qc0 = m.bf_qc0.as<int32_t>();
    a.qnc = m.bf_qnc.as<int32_t>(); a.qv = m.bf_qv.as<int32_t>(); a.vLa = m.bf_vLa.as<int32_t>();
    a.rtrace = m.bf_rtr.as<double>();
    QVTS_BF_PROF(m, 6, k_bf_backup<<<1, 256, 0, st>>>(a));
    QVTS_CUDA(cudaGetLastError());
    return QVTS_OK;
}

// node-pool arrays and their per-node element sizes (beliefs handled apart)
static void bf_pool_arrays(Model &m, std::vector<std::pair<DevBuf *, size_t>> &v) {
    v = {{&m.bf_path, 8}, {&m.bf_anc, 64}, {&m.bf_pq, 4}, {&m.bf_z, 4}, {&m.bf_f, 4}, {&m.bf_root, 4},
         {&m.bf_depth, 4}, {&m.bf_vE, 4}, {&m.bf_vq0, 4}, {&m.bf_vLa, 4}, {&m.bf_vU, 8}, {&m.bf_vL, 8},
         {&m.bf_vH, 8}, {&m.bf_qR, 8}, {&m.bf_qU, 8}, {&m.bf_qL, 8}, {&m.bf_qH, 8}, {&m.bf_qE, 4},
         {&m.bf_qc0, 4}, {&m.bf_qnc, 4}, {&m.bf_qv, 4}};
}

// grow every pool array to `cap` nodes keeping the first `used` (Q arrays: at most `used` too)
static qvts_status bf_pool_grow(Model &m, long long used, long long cap, cudaStream_t st) {
    std::vector<std::pair<DevBuf *, size_t>> arrs;
    bf_pool_arrays(m, arrs);
    arrs.push_back({&m.bf_bel, sizeof(float) * (size_t)m.HWp});
    for (auto &pr : arrs) {
        const size_t need = pr.second * (size_t)cap;
        if (pr.first->cap >= need) continue;
        DevBuf nb;
        QVTS_TRY(nb.ensure(need));
        if (used > 0 && pr.first->p)
            QVTS_CUDA(cudaMemcpyAsync(nb.p, pr.first->p, pr.second * (size_t)used, cudaMemcpyDeviceToDevice, st));
        QVTS_CUDA(cudaStreamSynchronize(st));
        pr.first->release();
        *pr.first = nb;
    }
    return QVTS_OK;
}

}  // namespace qvts

using namespace qvts;

extern "C" qvts_status qvts_plan_best_first(qvts_model *m, const float *root_dev, const qvts_bf_cfg *cfg,
                                            qvts_bf_result *res, void *stream) {
    qvts::NvtxRange nvtx_range__("qvts_plan_best_first");
    if (!m || !cfg || !res) { set_error("NULL argument"); return QVTS_ERR_INVALID_ARG; }
    if (cfg->n_samples < 1 || cfg->n_samples > 4096 || cfg->max_expansions < 0 || cfg->max_depth < 1 ||
        cfg->max_depth > 8 || !(cfg->gap_tol >= 0.0) ||
        (cfg->sampler != QVTS_SAMPLER_MARGINAL && cfg->sampler != QVTS_SAMPLER_ANCESTRAL)) {
        set_error("bad best-first config (n 1..4096, max_expansions >= 0, max_depth 1..8, gap_tol >= 0)");
        return QVTS_ERR_INVALID_ARG;
    }
    if (!m->have_fib) { set_error("run qvts_fib_iteration before best-first planning"); return QVTS_ERR_STATE; }
    if (!m->have_pbvi) { set_error("run qvts_pbvi before best-first planning"); return QVTS_ERR_STATE; }
    QVTS_CUDA(cudaSetDevice(m->device));
    // the work runs on a private non-blocking stream (a CUDA graph cannot be captured on the legacy
    // default stream), ordered after the caller's stream and before anything queued on it later
    cudaStream_t cst = (cudaStream_t)stream;
    if (!m->bf_stream) QVTS_CUDA(cudaStreamCreateWithFlags(&m->bf_stream, cudaStreamNonBlocking));
    if (!m->bf_join) QVTS_CUDA(cudaEventCreateWithFlags(&m->bf_join, cudaEventDisableTiming));
    QVTS_CUDA(cudaEventRecord(m->bf_join, cst));
    cudaStream_t st = m->bf_stream;
    QVTS_CUDA(cudaStreamWaitEvent(st, m->bf_join, 0));
    const auto t_start = std::chrono::steady_clock::now();
    const int NA = m->NA, HW = m->HW, n = cfg->n_samples;
    const BfGeom g = bf_geom(*m);
    const bool reuse = cfg->reuse && m->bf_valid;
    m->bf_valid = false;
    BfDev hs{};
    if (reuse) {   // keep pool fill and root; new limits below
        QVTS_CUDA(cudaMemcpyAsync(&hs, m->bf_sum.p, sizeof(BfDev), cudaMemcpyDeviceToHost, st));
        QVTS_CUDA(cudaStreamSynchronize(st));
        hs.root = m->bf_root_idx;
    } else {
        hs.depth = -1;
    }
    const long long used = reuse ? hs.nv : 0;
    // node pool: worst case used + 1 + max_expansions * per_exp nodes, allocated lazily in doublings
    // and capped at half the free device memory
    const long long per_exp = (long long)NA * std::min(n, 16);
    const long long worst = used + 1 + (long long)cfg->max_expansions * per_exp;
    size_t free_b = 0, total_b = 0;
    QVTS_CUDA(cudaMemGetInfo(&free_b, &total_b));
    const size_t node_bytes = (size_t)m->HWp * 4 + 200;
    auto pool_nodes = [&]() {   // nodes every pool array can hold now
        std::vector<std::pair<DevBuf *, size_t>> arrs;
        bf_pool_arrays(*m, arrs);
        arrs.push_back({&m->bf_bel, sizeof(float) * (size_t)m->HWp});
        long long c = LLONG_MAX;
        for (auto &pr : arrs) c = std::min(c, (long long)(pr.first->cap / pr.second));
        return c;
    };
    const long long have = m->bf_bel.p ? pool_nodes() : 0;
    const long long by_mem = std::max(used + 1 + per_exp, have + (long long)(free_b / 2 / node_bytes));
    const long long cap_max = std::min(worst, by_mem);
    long long cap = std::min(cap_max, used + 1 + 64 * per_exp);
    QVTS_TRY(bf_pool_grow(*m, used, cap, st));
    cap = std::min(cap_max, pool_nodes());
    const int nrows = g.nkb * g.KB;
    QVTS_TRY(m->bf_VT.ensure(sizeof(double) * (size_t)HW * nrows));
    QVTS_TRY(m->bf_part.ensure(sizeof(double) * (size_t)g.nkb * g.nsplit * 144 * g.KB));
    QVTS_TRY(m->bf_sum.ensure(sizeof(BfDev)));
    QVTS_TRY(m->bf_keys.ensure(sizeof(uint32_t) * 2));
    QVTS_TRY(m->bf_rtr.ensure(sizeof(double) * 2 * ((size_t)cfg->max_expansions + 1)));
    QVTS_TRY(bf_expand_prepare(*m, m->bf_ql, n, cfg->sampler));
    BfDev *S = m->bf_sum.as<BfDev>();
    hs.budget = cfg->max_expansions; hs.max_depth = cfg->max_depth; hs.per_exp = (int)per_exp;
    hs.gap_tol = cfg->gap_tol; hs.cap_v = cap;
    const long long nq0 = reuse ? hs.nq : 0;
    uint32_t keys[2] = {cfg->step, cfg->episode};
    QVTS_CUDA(cudaMemcpyAsync(m->bf_keys.p, keys, sizeof(keys), cudaMemcpyHostToDevice, st));
    QVTS_CUDA(cudaMemcpyAsync(S, &hs, sizeof(BfDev), cudaMemcpyHostToDevice, st));

    QVTS_CUDA(cudaEventRecord(m->ev0, st));
    k_bf_vk<<<(unsigned)(((long long)HW * nrows + 255) / 256), 256, 0, st>>>(m->d_alpha64.as<double>(), NA,
                                                                               m->pb_G.as<double>(), g.nal, HW, nrows,
                                                                               m->bf_VT.as<double>());
    if (reuse) {
        k_bf_resume<<<1, 1, 0, st>>>(S, m->bf_vE.as<int32_t>(), m->bf_depth.as<int32_t>(), m->bf_vU.as<double>(),
                                     m->bf_vL.as<double>(), m->bf_vH.as<double>(), m->bf_vLa.as<int32_t>(),
                                     m->bf_rtr.as<double>());
    } else {
        if (!root_dev) { set_error("root_dev is NULL without tree reuse"); return QVTS_ERR_INVALID_ARG; }
        QVTS_CUDA(cudaMemcpyAsync(m->bf_bel.p, root_dev, sizeof(float) * HW, cudaMemcpyDeviceToDevice, st));
        k_bf_init_root<<<1, 1, 0, st>>>(m->bf_path.as<uint64_t>(), m->bf_pq.as<int32_t>(), m->bf_z.as<int32_t>(),
                                        m->bf_f.as<int32_t>(), m->bf_root.as<int32_t>(), n);
        QVTS_CUDA(cudaGetLastError());
        QVTS_TRY(bf_leaf_bounds(*m, g, S, st));            // the root (S->depth = -1)
        k_bf_root_state<<<1, 1, 0, st>>>(S, m->bf_vU.as<double>(), m->bf_vL.as<double>(), m->bf_vH.as<double>(),
                                         m->bf_vLa.as<int32_t>(), m->bf_rtr.as<double>());
    }
    QVTS_CUDA(cudaGetLastError());
    // chunks of expansions replayed from a CUDA graph; the graph is re-captured after a pool growth
    // (the arrays move).  Profiling mode launches directly so every kernel is timed.
    const int chunk = 16;
    // the captured chunk depends only on the pool arrays and the by-value launch arguments: keep it
    // in the model and replay it on later calls while those are unchanged
    std::vector<uintptr_t> key;
    {
        std::vector<std::pair<DevBuf *, size_t>> arrs;
        bf_pool_arrays(*m, arrs);
        for (auto &pr : arrs) key.push_back((uintptr_t)pr.first->p);
        for (const DevBuf *b : {&m->bf_bel, &m->bf_VT, &m->bf_part, &m->bf_sum, &m->bf_keys, &m->bf_rtr, &m->part,
                                &m->counters, &m->xs, &m->bf_ql.R, &m->bf_ql.P, &m->bf_ql.cnt, &m->bf_ql.umask,
                                &m->bf_ql.U, &m->bf_ql.off, &m->bf_ql.Q})
            key.push_back((uintptr_t)b->p);
        for (long long v : {(long long)n, (long long)cfg->seed, (long long)cfg->sampler, (long long)g.XS,
                            (long long)g.nsplit, (long long)g.nvec, (long long)(uintptr_t)st})
            key.push_back((uintptr_t)v);
    }
    cudaGraphExec_t gexec = (m->bf_gexec && m->bf_gkey == key) ? m->bf_gexec : nullptr;
    auto capture = [&]() -> qvts_status {
        if (m->bf_gexec) { cudaGraphExecDestroy(m->bf_gexec); m->bf_gexec = nullptr; }
        gexec = nullptr;
        cudaGraph_t graph;
        QVTS_CUDA(cudaStreamBeginCapture(st, cudaStreamCaptureModeRelaxed));
        for (int i = 0; i < chunk; ++i) {
            const qvts_status s2 = bf_one_expansion(*m, g, S, *cfg, st);
            if (s2 != QVTS_OK) {
                cudaStreamEndCapture(st, &graph);
                return s2;
            }
        }
        QVTS_CUDA(cudaStreamEndCapture(st, &graph));
        const cudaError_t e = cudaGraphInstantiate(&gexec, graph, 0);
        cudaGraphDestroy(graph);
        QVTS_CUDA(e);
        m->bf_gexec = gexec;
        m->bf_gkey = key;
        return QVTS_OK;
    };
    const bool direct = m->prof;
    for (;;) {
        QVTS_CUDA(cudaMemcpyAsync(&hs, S, sizeof(BfDev), cudaMemcpyDeviceToHost, st));
        QVTS_CUDA(cudaStreamSynchronize(st));
        if (hs.done) break;
        if (cfg->time_budget_ms > 0.0 &&
            std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t_start).count() >=
                cfg->time_budget_ms) {
            hs.done = 1;
            hs.stop = QVTS_BF_TIME;
            break;
        }
        // room for a whole chunk, else grow (the device check stops at the pool limit)
        if (hs.nv + (long long)chunk * per_exp > cap && cap < cap_max) {
            const long long ncap = std::min(cap_max, std::max(2 * cap, hs.nv + (long long)chunk * per_exp));
            QVTS_TRY(bf_pool_grow(*m, hs.nv, ncap, st));
            cap = std::min(cap_max, pool_nodes());
            QVTS_CUDA(cudaMemcpyAsync(&S->cap_v, &cap, sizeof(long long), cudaMemcpyHostToDevice, st));
            QVTS_CUDA(cudaStreamSynchronize(st));
            // the arrays may have moved: the cached graph's key changes with them
            std::vector<std::pair<DevBuf *, size_t>> arrs;
            bf_pool_arrays(*m, arrs);
            for (size_t i = 0; i < arrs.size(); ++i) key[i] = (uintptr_t)arrs[i].first->p;
            key[arrs.size()] = (uintptr_t)m->bf_bel.p;
            if (key != m->bf_gkey) gexec = nullptr;
            // a growth (reallocation, copy) and the graph recapture it forces can take tens of
            // milliseconds: re-check the wall-clock budget before spending them on another chunk
            if (cfg->time_budget_ms > 0.0 &&
                std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t_start).count() >=
                    cfg->time_budget_ms) {
                hs.done = 1;
                hs.stop = QVTS_BF_TIME;
                break;
            }
        }
        if (direct) {
            for (int i = 0; i < chunk; ++i) QVTS_TRY(bf_one_expansion(*m, g, S, *cfg, st));
        } else {
            if (!gexec) QVTS_TRY(capture());
            QVTS_CUDA(cudaGraphLaunch(gexec, st));
        }
    }
    QVTS_CUDA(cudaEventRecord(m->ev1, st));
    QVTS_CUDA(cudaStreamSynchronize(st));
    QVTS_CUDA(cudaEventRecord(m->bf_join, st));
    QVTS_CUDA(cudaStreamWaitEvent(cst, m->bf_join, 0));
    const long long nv = hs.nv;
    const int nexp = hs.nexp;
    std::memset(res, 0, sizeof(*res));
    res->n_actions = NA;
    res->n_expansions = nexp;
    res->stop_reason = hs.stop;
    res->n_vnodes = nv;
    res->U = hs.U;
    res->L = hs.L;
    for (int j = 0; j < 9; ++j) res->u_q[j] = res->l_q[j] = NAN;
    int32_t rq0 = -1;   // the root's first Q-node (-1: unexpanded)
    QVTS_CUDA(cudaMemcpy(&rq0, m->bf_vq0.as<int32_t>() + hs.root, sizeof(int32_t), cudaMemcpyDeviceToHost));
    if (rq0 >= 0) {
        QVTS_CUDA(cudaMemcpy(res->u_q, m->bf_qU.as<double>() + rq0, sizeof(double) * NA, cudaMemcpyDeviceToHost));
        QVTS_CUDA(cudaMemcpy(res->l_q, m->bf_qL.as<double>() + rq0, sizeof(double) * NA, cudaMemcpyDeviceToHost));
    }
    float ms = 0.f;
    QVTS_CUDA(cudaEventElapsedTime(&ms, m->ev0, m->ev1));
    res->device_ms = ms;
    if (rq0 < 0) {
        res->action = m->pb_act[hs.la0];
    } else {                  // getOptimalAction: max L_Q, ties by U_Q then index
        int best = 0;
        for (int j = 1; j < NA; ++j)
            if (res->l_q[j] > res->l_q[best] || (res->l_q[j] == res->l_q[best] && res->u_q[j] > res->u_q[best])) best = j;
        res->action = m->action_id[best];
    }
    m->bf_nv = nv;
    m->bf_nq = hs.nq;
    m->bf_nq0 = nq0;
    m->bf_nexp = nexp;
    m->bf_root_idx = hs.root;
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
    if (exp_order) {   // Q-node blocks are allocated in expansion order: block e belongs to qv[e * NA]
        std::vector<int32_t> qv((size_t)m->bf_nq);
        if (m->bf_nq) QVTS_CUDA(cudaMemcpy(qv.data(), m->bf_qv.p, sizeof(int32_t) * qv.size(), cudaMemcpyDeviceToHost));
        for (int e = 0; e < m->bf_nexp; ++e) exp_order[e] = qv[(size_t)m->bf_nq0 + (size_t)e * m->NA];
    }
    if (root_trace)
        QVTS_CUDA(cudaMemcpy(root_trace, m->bf_rtr.p, sizeof(double) * 2 * ((size_t)m->bf_nexp + 1),
                             cudaMemcpyDeviceToHost));
    return QVTS_OK;
}

extern "C" qvts_status qvts_bf_advance(qvts_model *m, int32_t action, int32_t z, int32_t *reused, void *stream) {
    qvts::NvtxRange nvtx_range__("qvts_bf_advance");
    if (!m || !reused) { set_error("NULL argument"); return QVTS_ERR_INVALID_ARG; }
    *reused = 0;
    if (!m->bf_valid) { set_error("qvts_plan_best_first has not run"); return QVTS_ERR_STATE; }
    if (z < 0 || z > 15) { set_error("z must be 0..15"); return QVTS_ERR_INVALID_ARG; }
    int j = -1;
    for (int k = 0; k < m->NA; ++k) if (m->action_id[k] == action) j = k;
    if (j < 0) { set_error("action is not in the model's action set"); return QVTS_ERR_INVALID_ARG; }
    QVTS_CUDA(cudaSetDevice(m->device));
    cudaStream_t st = (cudaStream_t)stream;
    QVTS_CUDA(cudaStreamSynchronize(m->bf_stream));
    const int r = m->bf_root_idx;
    int32_t q0 = -1;
    QVTS_CUDA(cudaMemcpy(&q0, m->bf_vq0.as<int32_t>() + r, sizeof(int32_t), cudaMemcpyDeviceToHost));
    if (q0 < 0) return QVTS_OK;                     // unexpanded root: nothing to keep
    int32_t c0 = 0, nc = 0;
    QVTS_CUDA(cudaMemcpy(&c0, m->bf_qc0.as<int32_t>() + q0 + j, sizeof(int32_t), cudaMemcpyDeviceToHost));
    QVTS_CUDA(cudaMemcpy(&nc, m->bf_qnc.as<int32_t>() + q0 + j, sizeof(int32_t), cudaMemcpyDeviceToHost));
    std::vector<int32_t> zs(std::max(1, nc));
    if (nc > 0) QVTS_CUDA(cudaMemcpy(zs.data(), m->bf_z.as<int32_t>() + c0, sizeof(int32_t) * nc, cudaMemcpyDeviceToHost));
    int c = -1;
    for (int i = 0; i < nc; ++i) if (zs[i] == z) c = c0 + i;
    if (c < 0) return QVTS_OK;                      // z was not sampled: the caller starts afresh
    const long long nv = m->bf_nv;
    k_bf_rebase<<<(unsigned)((nv + 255) / 256), 256, 0, st>>>(nv, c, m->bf_path.as<uint64_t>(), m->bf_depth.as<int32_t>(),
                                                             m->bf_anc.as<int32_t>(), m->bf_pq.as<int32_t>());
    QVTS_CUDA(cudaGetLastError());
    QVTS_CUDA(cudaStreamSynchronize(st));
    m->bf_root_idx = c;
    *reused = 1;
    return QVTS_OK;
}
