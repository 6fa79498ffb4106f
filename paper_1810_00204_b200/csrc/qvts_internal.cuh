// qvts_internal.cuh — internal structures of libqvts (not part of the ABI).
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <string>
#include <vector>

#include "../../include/qvts.h"

#include <nvtx3/nvToolsExt.h>

namespace qvts {

// NVTX range for the duration of a scope (ABI entry points, plan-step levels): visible in Nsight
// Systems / Compute timelines, a no-op without an attached tool (SURVEY §5 tracing)
struct NvtxRange {
    explicit NvtxRange(const char *name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
    NvtxRange(const NvtxRange &) = delete;
    NvtxRange &operator=(const NvtxRange &) = delete;
};

constexpr int kHistThreads = 128;   // slot-threads per band list (one class stream per slot-thread)
constexpr int kPairThreads = 256;   // hist CTA: 2 parents x 128 slot-threads
constexpr int kMaxLevels = 9;       // depth <= 8

void set_error(const std::string &msg);

#define QVTS_CUDA(call)                                                                   \
    do {                                                                                  \
        cudaError_t e__ = (call);                                                         \
        if (e__ != cudaSuccess) {                                                         \
            ::qvts::set_error(std::string(#call) + ": " + cudaGetErrorString(e__));       \
            return e__ == cudaErrorMemoryAllocation ? QVTS_ERR_OUT_OF_MEMORY : QVTS_ERR_CUDA; \
        }                                                                                 \
    } while (0)

#define QVTS_TRY(expr)                          \
    do {                                        \
        qvts_status s__ = (expr);               \
        if (s__ != QVTS_OK) return s__;         \
    } while (0)

// Growable device buffer (capacity only grows; contents are not preserved on growth).
struct DevBuf {
    void *p = nullptr;
    size_t cap = 0;
    qvts_status ensure(size_t bytes);
    void release();
    template <class T> T *as() const { return static_cast<T *>(p); }
};

// Page-locked host staging (cudaHostAlloc): small per-call uploads and readbacks run as true
// asynchronous copies instead of staged pageable ones
struct HostBuf {
    void *p = nullptr;
    size_t cap = 0;
    qvts_status ensure(size_t bytes);
    void release();
    template <class T> T *as() const { return static_cast<T *>(p); }
};

// One row band of the grid processed by one hist CTA: rows [row0, row0+nrows), with a
// class-partitioned slot list (SURVEY §7 "signature binning": every thread owns a stream of
// cells that share one wall signature, so its bin index is fixed in registers).
struct BandInfo {
    int row0, nrows, L, pad;
    long long slot_off;           // first slot; slot (i, t) = slot_off + i*kHistThreads + t
    int cs[17];                   // threads [cs[c], cs[c+1]) own class c; >= cs[16] idle
    int pad2[3];
};

struct BandSet {
    int nb = 0, rows = 0, tile_floats = 0, tile_pitch = 0;   // tile column c at c + 4
    long long total_slots = 0;
    std::vector<BandInfo> h_bands;
    std::vector<int32_t> h_slot_cell;
    DevBuf bands, entries, slot_cell, qlist, qlist_fib;
};

// Leaf level (leaf.cu): one CTA of kLeafThreads slot-threads per PAIR of leaf parents walks every
// row band of the grid; slot-thread t owns wall-signature class cls(t) in every band (class slot
// ranges fixed for the whole grid), so its fp32 accumulators run across all bands and the class
// reduction happens once per parent pair: one fp64 partial record per parent (per band group).
constexpr int kLeafThreads = 128;
struct LeafBand {
    int row0, nrows, L, pad;      // L = steps of this band (multiple of 4); entries padded by 8 more steps
    long long slot_off;           // slot (i, t) of this band = slot_off + i * kLeafThreads + t
};
struct LeafBands {
    int nb = 0, rows = 0, TP = 0, TS = 0;   // segment row pitch; one parent's tile (all segments), floats
    int nseg = 1, SW = 0, HB = 0;            // column segments of SW cells (grid column c of segment s at
                                             // c - s SW + 4 of its rows), segment stride HB
    int cs[17] = {0};                        // slot-threads [cs[c], cs[c+1]) own class c in every band
    long long total_slots = 0, steps = 0;    // steps = sum of the bands' L (padding included)
    std::vector<LeafBand> h_bands;
    std::vector<int32_t> h_slot_cell;
    DevBuf bands, entries, slot_cell, qlist, qlist_fib;
};

// Tensor-core leaf level (leafmma.cu): per row band, the free cells sorted by wall-signature class
// and cut into chunks of 16 (the MMA's K); per (chunk, lane) the Q' B fragments.
struct LeafMma {
    int R = 0, nb = 0, TP = 0, tile_words = 0, ptile = 0;   // nb = 0: not available (scalar leaf kernel)
    long long nchunks = 0;
    std::vector<int32_t> h_cs;       // [nb][17] chunk ranges per class (host only)
    std::vector<int32_t> h_cells;    // [nchunks][16] cell of each K position (-1 = padding)
    DevBuf wr;                       // [nb][5] chunk range of each warp quarter in the band
    DevBuf offs;                     // [nchunks][4] uint4: byte offsets of a lane's 4 cells, class << 28
    DevBuf dmask;                    // [nchunks][4] uint4: per diagonal, byte e = 0x80 if occ(cell e + d_k)
    DevBuf cells;                    // [nchunks][16] (h_cells on the device, for the fragment build)
    DevBuf qfr, qfr_fib;             // [nchunks][32] uint4 B fragments of Q' (Q_MDP / FIB leaves)
};

// Per-level node arrays of the level-batched tree (SoA).
struct VLevel {
    long long n = 0;                  // V-nodes at this level
    DevBuf path, parent_q, z, f, root, V, belief;
};
struct QLevel {
    long long nwork = 0;              // parents expanded at this level (owned subset when sharded)
    DevBuf vmap;                      // work index -> V-node index (only when sharded)
    bool mapped = false;
    const int32_t *vmap_ptr = nullptr;   // the map in use (vmap, or the caller's active-root list)
    DevBuf R, P, cnt, umask, U, off, Q, zdraw, leafV, xdraw;
};

struct Model {
    int device = 0;
    int H = 0, W = 0, HW = 0, HWp = 0, NA = 0, NAP = 0, goal = 0;
    uint32_t mask = 0;
    int action_id[9] = {0};
    double p_int = 0, p_stay = 0, p_lat = 0, acc = 0, gamma = 0;
    std::vector<uint8_t> occ, m8, sig;
    std::vector<double> R64;          // [NA][HW]
    // device tables
    DevBuf d_m8, d_sig, d_cell /* sig | occ<<4 */, d_ctab, d_R64, d_O64, d_O32, d_gc_cell, d_gc_off /* [NA+1] per-action ranges */, d_gc_val, d_free;
    int ngc = 0;
    BandSet band_big, band_small;
    LeafBands leafb;
    LeafMma lm;
    // value iteration
    bool have_q = false;
    double qbar = 0.0;
    DevBuf d_V[2], d_resid, d_Q64;
    // Fast Informed Bound (NEXT-1)
    bool have_fib = false;
    double qbar_fib = 0.0;
    DevBuf d_A[2], d_alpha64;
    int cur_leaf = 0;                 // leaf alpha-set of the plan being built (qvts_leaf_bound)
    // plan workspace
    VLevel vl[kMaxLevels + 1];
    QLevel ql[kMaxLevels];
    DevBuf part, scan_tmp, total, counters, vshard, xs;
    int last_depth = -1, last_n = 0, last_shard_level = -1;
    long long last_flagged = 0, last_skipped = 0;
    bool last_xdraws = false;
    bool last_trace = false;
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;
    // graph-captured plan step (small trees): device level counts, private stream, cached graph
    DevBuf lvl_cnt, root_buf;
    cudaStream_t pg_stream = nullptr;
    cudaEvent_t pg_join = nullptr;
    cudaGraphExec_t pg_exec = nullptr;
    std::vector<uintptr_t> pg_key;
    // instrumentation
    bool prof = false;
    qvts_profile pstat{};
    std::vector<cudaEvent_t> evpool;
    struct EvRec { int cat; cudaEvent_t a, b; };
    std::vector<EvRec> evrecs;
    size_t evnext = 0;
    long long n_free = 0;
    // belief_update scratch
    DevBuf bu_R, bu_P, bu_cnt, bu_umask, bu_U, bu_off, bu_path, bu_root;
    HostBuf bu_host;                            // qvts_belief_update_batch's selection upload / P readback
    // episodes
    DevBuf ep_b[2], ep_state, ep_root_step, ep_root_ep;
    // PBVI lower bound (NEXT-2, pbvi.cu)
    bool have_pbvi = false;
    int pb_np = 0, pb_nal = 0, pb_P = 0;
    std::vector<int32_t> pb_act;
    DevBuf pb_b0, pb_B, pb_G, pb_Gn, pb_GT, pb_Bbar, pb_Sc, pb_Rb, pb_sel, pb_astar, pb_cand, pb_misc, pb_cls, pb_chunks,
        pb_part;
    // anytime best-first QVTS (NEXT-2, bestfirst.cu): node pool of the last qvts_plan_best_first
    bool bf_valid = false;
    long long bf_nv = 0, bf_nq = 0, bf_nq0 = 0;
    int bf_nexp = 0, bf_root_idx = 0;
    DevBuf bf_bel, bf_path, bf_pq, bf_z, bf_f, bf_root, bf_depth, bf_vU, bf_vL, bf_vH, bf_vE, bf_vq0, bf_vLa;
    DevBuf bf_qR, bf_qU, bf_qL, bf_qH, bf_qE, bf_qc0, bf_qnc, bf_qv;
    DevBuf bf_VT, bf_part, bf_sum, bf_keys, bf_anc, bf_rtr;
    cudaStream_t bf_stream = nullptr;
    cudaGraphExec_t bf_gexec = nullptr;          // cached chunk graph and its key
    std::vector<uintptr_t> bf_gkey;
    cudaEvent_t bf_join = nullptr;
    QLevel bf_ql;
};

// instrumentation helpers (model.cu)
void prof_begin(Model &m, int cat, cudaStream_t st, cudaEvent_t *out);
void prof_end(Model &m, int cat, cudaStream_t st, cudaEvent_t a);
void prof_collect(Model &m);   // after a stream sync: fold recorded event pairs into pstat

template <class T>
static qvts_status upload(DevBuf &b, const std::vector<T> &v) {
    QVTS_TRY(b.ensure(sizeof(T) * (v.size() > 1 ? v.size() : 1)));
    if (!v.empty()) QVTS_CUDA(cudaMemcpy(b.p, v.data(), sizeof(T) * v.size(), cudaMemcpyHostToDevice));
    return QVTS_OK;
}

// leafmma.cu
qvts_status build_leaf_mma(Model &m);
qvts_status build_leaf_qfrag(Model &m, const double *src64, double qbar, bool fib, cudaStream_t st);
bool leaf_mma_enabled(const Model &m, long long bstride, const float *beliefs);
int leaf_mma_records();              // fp64 records per parent written by the leaf kernel (one per warp)
qvts_status launch_leaf_mma(Model &m, const float *beliefs, long long bstride, const int32_t *vmap, long long nwork,
                            int pstride, cudaStream_t st, const int32_t *skip, const long long *nwork_dev);

// leaf.cu: the class-fixed band lists, and the leaf-level launch (S1+S2+S5 for every leaf parent);
// nsplit CTAs share a parent pair's bands (one fp64 record each, summed in split order by k_reduce)
qvts_status build_leaf_bands(Model &m, LeafBands &lb);
bool leaf_kernel_supported(const Model &m);
int leaf_nsplit(const Model &m, int level);
qvts_status launch_leaf(Model &m, const float *beliefs, long long bstride, long long nbel, const int32_t *vmap,
                        long long nwork, int nsplit, int pstride, long long part_off, cudaStream_t st,
                        const long long *nwork_dev = nullptr);

// model.cu
qvts_status build_bands(Model &m, BandSet &bs, int rows);
qvts_status build_qlists(Model &m, const double *src64, double qbar, bool fib, cudaStream_t st);

// plan.cu
struct RootBatch {
    const float *beliefs;       // [n][stride]
    long long stride;
    long long n;
    const uint32_t *step_dev;   // [n] per-root step keys (device)
    const uint32_t *episode_dev;// [n] per-root episode keys (device)
    const int32_t *active = nullptr;   // optional: expand only these roots (device [n_active])
    long long n_active = 0;
};
qvts_status plan_levels(Model &m, const RootBatch &roots, const qvts_plan_cfg &cfg, const qvts_comm *comm,
                        cudaStream_t st, long long *nv_out /*[depth+1]*/);
// P(z|b,a) and R(b,a) of the (active) roots only, into ql[0] (S1+S2 without sampling)
qvts_status root_marginals(Model &m, const RootBatch &roots, cudaStream_t st);
// Explicit V-node batch of one level (best-first QVTS): S1-S3 + child offsets, then S4.
struct ExpandSpec {
    const float *beliefs;
    long long bstride, nwork;
    const uint64_t *vpath;
    const int32_t *vroot;
    const uint32_t *root_step, *root_ep;
    int level, n;
    uint32_t seed;
    int sampler;
};
struct ChildOut {
    float *belief;
    long long stride;
    uint64_t *path;
    int32_t *parent_q, *z, *f, *root;
};
qvts_status expand_marginals(Model &m, const ExpandSpec &e, QLevel &ql, cudaStream_t st, long long *total);
// Graph-capturable best-first expansion (bestfirst.cu): indices read from device memory.
struct BfLaunch {
    float *bel;                       // node pool beliefs [cap][stride]
    long long stride;
    uint64_t *path;
    int32_t *pq, *z, *f, *root;
    const int32_t *sel, *skip;        // node to expand; non-zero = planning finished
    const long long *cbase;           // first free pool slot
    long long *total;                 // out: children of this expansion
    const uint32_t *root_step, *root_ep;
    int n;
    uint32_t seed;
    int sampler;
};
qvts_status bf_expand_prepare(Model &m, QLevel &ql, int n, int sampler);
qvts_status bf_expand_launch(Model &m, const BfLaunch &L, QLevel &ql, cudaStream_t st);
qvts_status expand_children(Model &m, const ExpandSpec &e, const QLevel &ql, const ChildOut &o, cudaStream_t st);
// Bayes correction of selected (Q-node, z) pairs of level 0 into out[sel_out[g]*ostride]
qvts_status correct_selected(Model &m, const RootBatch &roots, const int32_t *sel_q, const int32_t *sel_z,
                             const int32_t *sel_out, long long n, float *out, long long ostride, cudaStream_t st);

}  // namespace qvts

struct qvts_model : public qvts::Model {};
