/* qvts.h — C ABI of the B200-native QV-Tree Search hot path (libqvts.so).
 *
 * Paper: "QV-Tree Search" (arXiv 1810.00204); citations are PAPER.md lines of that paper's
 * source, plus the reading numbers R1..R35 of SURVEY.md §8(c) c.3 restated in DESIGN.md.
 *
 * General conventions (every entry point):
 *  - All functions are extern "C" and return qvts_status (QVTS_OK = 0) unless void.  On failure
 *    qvts_last_error() returns a thread-local, human-readable message for the last failure.
 *  - A qvts_model handle owns its device tables and workspace on ONE CUDA device (the one
 *    named in the descriptor).  One handle is used by one host thread at a time.
 *  - `stream` is a cudaStream_t passed as void* (NULL = the legacy default stream).  Work is
 *    enqueued on it; calls that return host values synchronise it before returning.
 *  - Caller buffers: "_dev" pointers are device memory on the model's device, fp32, contiguous
 *    H*W cells in row-major order (cell i = r*W + c, row 0 = top),
 *    4-byte aligned; "_host" pointers are host memory.  The caller owns every buffer it passes
 *    and the library never retains one after the call returns.
 *  - Actions are identified by their stencil id a = 3(dr+1) + (dc+1) in 0..8, where 4 = stay
 *    ("N_4(x) = x").  Arrays indexed "by action" list the model's action set in
 *    ascending stencil id.  Observations z are 4-bit words 0..15, bit k = sensor N_{2k+1}
 *    (bit0 up, bit1 left, bit2 right, bit3 down, reading R6).
 *  - Beliefs passed in must be non-negative, zero on occupied cells and sum to 1 (± 1e-4).
 *    Occupied cells are absorbing with no mass (R5); the kernels rely on those zeros (e.g. the
 *    batched update multiplies them by a zero weight instead of testing the occupancy).
 */
#ifndef QVTS_H
#define QVTS_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#if defined(__GNUC__)
#define QVTS_API __attribute__((visibility("default")))
#else
#define QVTS_API
#endif

typedef enum {
    QVTS_OK = 0,
    QVTS_ERR_INVALID_ARG = 1,     /* a pointer, index, size or config value is out of range   */
    QVTS_ERR_INVALID_MODEL = 2,   /* descriptor violates the model invariants */
    QVTS_ERR_STATE = 3,           /* call order violated (e.g. plan before value iteration)   */
    QVTS_ERR_NOT_CONVERGED = 4,   /* value iteration hit max_sweeps; last iterate is kept     */
    QVTS_ERR_ZERO_LIKELIHOOD = 5, /* P(z|b,a) <= 1e-30 in belief_update (R25)     */
    QVTS_ERR_OUT_OF_MEMORY = 6,   /* device allocation failed; the handle stays usable        */
    QVTS_ERR_CUDA = 7,            /* a CUDA runtime error; see qvts_last_error()              */
    QVTS_ERR_COMM = 8             /* the multi-rank all-reduce callback returned non-zero     */
} qvts_status;

typedef struct qvts_model qvts_model;   /* opaque */

/* ---- (1) model ------------------------------------------------------------------------
 * The POMDP tuple (X, A, Z, T, O, R, b0, gamma) of PAPER.md:44, compiled from an occupancy
 * grid per §V:
 *   T: 3x3 stencil, T'(x,a,N_a)=p_intended, T'(x,a,x)=p_stay, p_lateral on the two ring
 *      neighbours of N_a (readings R1-R3); stay deterministic; mass on occupied or off-map
 *      cells is accumulated to x (R4).
 *   O: 4 wall sensors on N1,N3,N5,N7, each correct with probability sensor_acc.
 *   R: r(y) = -2 occupied/off-map, 0 goal, -1 otherwise; R(x,4) = -2 off goal, otherwise
 *      R(x,a) = sum_y r(y) T'(x,a,y) with the pre-clamp T'.          */
typedef struct {
    int32_t height, width;         /* grid size; height*width <= 2^22                          */
    const uint8_t *occupancy;      /* host, height*width bytes, non-zero = occupied; copied     */
    int32_t goal;                  /* goal cell index; must be free                             */
    uint32_t action_mask;          /* bit a => stencil action a in A.  Supported sets:          */
                                   /* 0x1FF (A9, paper), 0x1EF (A8), 0x0AA (A4) (reading R19)   */
    double p_intended, p_stay, p_lateral;  /* >= 0, p_int + p_stay + 2 p_lat = 1 +- 1e-9      */
    double sensor_acc;             /* in (0.5, 1]; paper 0.95                                   */
    double gamma;                  /* in (0, 1); default 0.95 (reading R8)                      */
    int32_t device;                /* CUDA device ordinal                                       */
} qvts_model_desc;

/* Validate and compile the model, upload its tables.  No device compute.  Errors:
 * QVTS_ERR_INVALID_MODEL (descriptor invariants), QVTS_ERR_INVALID_ARG (unsupported
 * action_mask, NULL pointers), QVTS_ERR_CUDA / QVTS_ERR_OUT_OF_MEMORY.  *out is NULL on error. */
QVTS_API qvts_status qvts_model_create(const qvts_model_desc *desc, qvts_model **out);
QVTS_API void qvts_model_destroy(qvts_model *model);                     /* NULL is a no-op */
QVTS_API const char *qvts_last_error(void);

/* Number of actions and their stencil ids (ascending), and the cell count H*W. */
QVTS_API qvts_status qvts_model_info(const qvts_model *model, int32_t *n_actions, int32_t *action_ids /*[9]*/,
                            int64_t *n_cells);
/* Host copies of the compiled tables for table-parity tests: R as fp32 [|A|][H*W] and the
 * 4-bit wall signature sig(x) [H*W] (Appendix B.5).  Either pointer may be NULL. */
QVTS_API qvts_status qvts_model_tables(const qvts_model *model, float *R_host, uint8_t *sig_host);

/* ---- (2) offline MDP value iteration (reading R24) -----------------------
 * Synchronous Jacobi in fp64 from V0 = 0: V_{k+1}(x) = max_a [R(x,a) + gamma sum_y
 * T(x,a,y) V_k(y)], stopping at the first sweep with max_x |V_{k+1} - V_k| < eps; then
 * Q(x,a) = R + gamma T V.  Occupied cells: V = Q = 0.  The result (Q_MDP, the leaf alpha-vectors
 * of Eq. 4 with one vector per action, reading R14) is kept on the device for plan steps.
 * Returns QVTS_ERR_NOT_CONVERGED (Q still produced from the last iterate) if max_sweeps runs out. */
QVTS_API qvts_status qvts_value_iteration(qvts_model *model, double eps, int32_t max_sweeps,
                                 int32_t *sweeps_out, double *residual_out, void *stream);
/* Host copy of Q in fp64, layout [|A|][H*W]; QVTS_ERR_STATE before value iteration. */
QVTS_API qvts_status qvts_get_q(const qvts_model *model, double *q_host);

/* ---- (2b) Fast Informed Bound (Eq. 6-7) ------------
 * alpha^a(x) = R(x,a) + gamma sum_z max_a' sum_x' O(x',z) T(x,a,x') alpha^a'(x'), synchronous
 * fp64 iteration from alpha = max R / (1 - gamma) to max|delta| < eps.  The result
 * is one alpha-vector per action, an upper bound on V* no looser than Q_MDP; plan steps with
 * cfg.leaf_bound = QVTS_LEAF_FIB score leaves with it (Eq. 4).  Occupied cells: alpha = 0. */
QVTS_API qvts_status qvts_fib_iteration(qvts_model *model, double eps, int32_t max_sweeps,
                                        int32_t *sweeps_out, double *residual_out, void *stream);
/* Host copy of alpha_FIB in fp64, [|A|][H*W]; QVTS_ERR_STATE before qvts_fib_iteration. */
QVTS_API qvts_status qvts_get_alpha(const qvts_model *model, double *alpha_host);

/* ---- (2c) PBVI lower bound (§IV-B), fp64 ---------
 * Belief set: starts at {b0} (b0_dev: device fp32 [H*W], or NULL = uniform over free cells);
 * `expansions` rounds, each visiting the points present at its start in order: one Alg. 4 sample
 * per action (Philox4x32-10 ctr = (action index, point, round, 0x7BB1), key = (seed, 0xB5E7),
 * words 1..3 = x ~ b, x' ~ T, z ~ O), the Bayes posterior of each, and the one farthest in L1
 * from the set as grown so far is appended if that distance is > 0 (ties: lowest action index;
 * zero-likelihood posteriors skipped); stops at max_points (1..1024).
 * Backups: Gamma = {R_min / (1 - gamma)} (R_min over free cells and actions), then `sweeps`
 * point-based backups; each gives every point b the vector
 * alpha_b = R(.,a*) + gamma sum_z g_{a*,z}^{alpha*_{a*,z}}, alpha* = argmax_alpha b . g, a* = argmax of
 * the backed-up value (ties: lowest index).  Occupied cells: alpha = 0.  Synchronises `stream`;
 * *n_points_out = the number of belief points (= alpha vectors after >= 1 sweep). */
QVTS_API qvts_status qvts_pbvi(qvts_model *model, const float *b0_dev, int32_t expansions, int32_t max_points,
                               uint32_t seed, int32_t sweeps, int32_t *n_points_out, void *stream);
/* Host copies after qvts_pbvi (any pointer may be NULL): points fp64 [n_points][H*W], alpha fp64
 * [n_alpha][H*W], actions int32 [n_points] (stencil ids; 0 before any sweep); QVTS_ERR_STATE
 * before qvts_pbvi. */
QVTS_API qvts_status qvts_get_pbvi(const qvts_model *model, double *points_host, double *alpha_host,
                                   int32_t *actions_host, int32_t *n_alpha_out);

/* ---- (3) Bayes belief update, Eq. 3 ----------------------------------
 * out(x') = O(x',z) sum_x T(x,a,x') b(x) / P(z|b,a); *p_obs_out = P(z|b,a) (fp64).
 * b_dev and out_dev: device fp32 [H*W] (may not alias).  QVTS_ERR_ZERO_LIKELIHOOD when
 * P(z|b,a) <= 1e-30 (out_dev is then left unspecified).  Synchronises `stream`. */
QVTS_API qvts_status qvts_belief_update(qvts_model *model, const float *b_dev, int32_t action, int32_t z,
                               float *out_dev, double *p_obs_out, void *stream);

/* Batched Eq. 3 (SURVEY d.3 K9 at HBM scale): out_g = Phi(b_g, actions[g], zs[g]) for g < n.
 * b_dev: device fp32 [n][b_stride] (b_stride >= H*W floats), out_dev: device fp32 [n][out_stride]
 * (may not alias b_dev); actions (stencil ids) and zs: host int32 [n]; p_obs_out: host fp64 [n]
 * or NULL.  Two passes over each belief: P(z|b,a) = sum_x' O(x',z) bbar_a(x') for the selected
 * (a, z) only, then the correction (k_correct).  QVTS_ERR_ZERO_LIKELIHOOD if any P(z_g|b_g,a_g) <= 1e-30 (those
 * outputs unspecified, the rest valid).  Synchronises `stream`. */
QVTS_API qvts_status qvts_belief_update_batch(qvts_model *model, const float *b_dev, int64_t b_stride, int32_t n,
                                              const int32_t *actions, const int32_t *zs, float *out_dev,
                                              int64_t out_stride, double *p_obs_out, void *stream);

/* ---- (4) plan step: level-batched QV-tree expansion (Alg. 1-7) --------
 * Expands every V-node of a level at once, for depth levels 0..depth-1: predict through T,
 * marginal P(z|b,a) and R(b,a), n forward-sampled observations per Q-node from Philox4x32-10
 * keyed ctr = (sample j, path_lo, path_hi, step), key = (seed, episode) (SURVEY Appendix A,
 * readings R9/R10), one child per unique z weighted by its frequency f/n,
 * Q_MDP leaves (Eq. 4, R14), backup Q = R + gamma sum (f/n) V, V = max_a Q (Alg. 6-7, R13),
 * action = argmax_a Q(root, a), ties to the lowest stencil id (R16/R18). */
typedef enum { QVTS_LEAF_QMDP = 0, QVTS_LEAF_FIB = 1 } qvts_leaf_bound;
/* Observation sampler: the marginal draw z ~ P(z|b,a) on Philox word 0 (reading R9, default), or
 * Alg. 4 literally: x ~ b on word 1 (fp64 prefix sums over the grid),
 * x' ~ T(x,a,.) on word 2 (clamped row in stencil order, blocked targets merged into the stay
 * entry at first occurrence), z ~ O(x',.) on word 3. */
typedef enum { QVTS_SAMPLER_MARGINAL = 0, QVTS_SAMPLER_ANCESTRAL = 1 } qvts_sampler;
typedef struct {
    int32_t depth;        /* number of action levels D, 1..8 (reading R15)                       */
    int32_t n_samples;    /* observations drawn per Q-node, 1..4096                               */
    uint32_t seed, step, episode;
    int32_t want_trace;   /* 1: keep per-node draws for qvts_trace_* (costs memory)               */
    int32_t leaf_bound;   /* qvts_leaf_bound: Q_MDP (north star, R14) or FIB (needs qvts_fib_iteration) */
    int32_t sampler;      /* qvts_sampler                                                          */
} qvts_plan_cfg;

typedef struct {
    int32_t action;               /* chosen stencil id                                         */
    int32_t n_actions;
    double q_root[9];             /* Q(root, a) for the model's actions, ascending stencil id  */
    int64_t n_vnodes[9];          /* V-nodes per level 0..depth (level 0 = root = 1)           */
    int64_t n_belief_updates;     /* sum of n_vnodes[1..depth] created by this call (SURVEY d.2) */
    double device_ms;             /* CUDA-event time of the whole step on `stream`             */
    int32_t shard_level;          /* multi-rank: first rank-local level is shard_level+1; -1 none */
    int64_t n_flag_candidates;    /* draws of this step whose u * C_15 lies within 1e-6 of a boundary
                                     of the GPU's own fp64 CDF (the c.5 "flagged" draws; marginal
                                     sampler; on a rank: its own Q-nodes only)                  */
    int64_t n_tiles_skipped;      /* (parent pair, row band) tiles whose beliefs held no mass and
                                     were skipped (active-tile skipping)    */
} qvts_plan_result;

/* Multi-rank plan step: levels above `shard_level` are replicated, the V-nodes
 * of shard_level with canonical index i are expanded by rank i % nranks only, and the
 * zero-padded fp64 array of their values is summed across ranks by `allreduce_sum_f64`
 * (in place, on device memory, on `stream`; return 0 on success) — exact, so the root action
 * and Q are bit-identical for any rank count.  Pass NULL for a single GPU. */
typedef struct {
    int32_t rank, nranks;
    int32_t min_nodes_per_rank;   /* shard at the first level with >= this * nranks V-nodes */
    int (*allreduce_sum_f64)(void *ctx, double *buf_dev, int64_t count, void *stream);
    void *ctx;
} qvts_comm;

/* root_dev: device fp32 [H*W] belief (caller-owned).  Requires value iteration first
 * (QVTS_ERR_STATE).  QVTS_ERR_OUT_OF_MEMORY when the tree does not fit; the handle stays usable.
 * Synchronises `stream` (the host reads one child count per level and the root values). */
QVTS_API qvts_status qvts_plan_step(qvts_model *model, const float *root_dev, const qvts_plan_cfg *cfg,
                           const qvts_comm *comm, qvts_plan_result *result, void *stream);

/* ---- instrumentation (bench.py roofline) ----------------------------------------------
 * When enabled, every kernel launch of plan steps is bracketed by CUDA events on the launching
 * stream and its duration accumulated per kernel class: 0 leaf hist (S1+S2+S5), 1 hist (S1+S2),
 * 2 leaf reduce/sample (S2 tail+S3+S5 tail), 3 reduce/sample, 4 scan, 5 correct (S4),
 * 6 backup (S6), 7 other.  leaf_cells = sum over leaf-hist launches of parents x free cells. */
typedef struct {
    int64_t launches[8];
    double ms[8];
    int64_t leaf_cells, hist_cells, correct_cells_written;
    int64_t total_launches;       /* every kernel the library launched since the last reset   */
} qvts_profile;
QVTS_API qvts_status qvts_set_profiling(qvts_model *model, int32_t enable);   /* also resets */
QVTS_API qvts_status qvts_get_profile(const qvts_model *model, qvts_profile *out);

/* ---- plan trace (the last plan step of this handle; valid until the next plan step) ------
 * Levels: V-nodes exist at levels 0..D (0 = root), Q-nodes at levels 0..D-1; Q-node index
 * q = v*|A| + k for the k-th action of V-node v of the same level.  Children of a Q-node are
 * contiguous at the next V-level in ascending z.  Leaf V-nodes (level D) are not materialised:
 * their values are read with qvts_trace_leaf_values.  Beliefs exist for levels 0..D-1. */
QVTS_API qvts_status qvts_trace_qnodes(const qvts_model *model, int32_t level, uint64_t *path, double *R,
                              double *P /*[n][16]*/, uint16_t *cnt /*[n][16]*/, double *Q,
                              uint8_t *z /*[n][n_samples] or NULL; needs want_trace*/);
QVTS_API qvts_status qvts_trace_vnodes(const qvts_model *model, int32_t level, uint64_t *path,
                              int32_t *parent_q, int32_t *zobs, int32_t *freq, double *V);
/* Leaf values of the last Q-level, [n_q(D-1)][16] (entries for unsampled z are 0). */
QVTS_API qvts_status qvts_trace_leaf_values(const qvts_model *model, double *V /*[n][16]*/);
/* Levels of the last plan step: *depth, V-node counts n_v[0..depth-1] (materialised levels) and
 * the number of expanded V-nodes n_qwork[0..depth-1] per Q-level (n_q = n_qwork * |A|). */
QVTS_API qvts_status qvts_trace_counts(const qvts_model *model, int32_t *depth, int64_t *n_v, int64_t *n_qwork);
QVTS_API qvts_status qvts_trace_belief(const qvts_model *model, int32_t level, int64_t index, float *out_host);
/* Alg. 4 sampler (QVTS_SAMPLER_ANCESTRAL) with want_trace: the state index x of every draw,
 * [n_q][n_samples] int32 (row-major cell index), level 0..D-1.  QVTS_ERR_STATE otherwise. */
QVTS_API qvts_status qvts_trace_state_draws(const qvts_model *model, int32_t level, int32_t *x);

/* ---- (4b) anytime best-first QVTS (Alg. 1 inner loop + Algs. 2-7, Eq. 8; PAPER.md:130-298;
 * SURVEY §8(f) NEXT-2; reading B5) -------------------------------------------------
 * Tree s = QVSearchTree(b0): one leaf with U = V_FIB(b0), L = V_PBVI(b0), H = U - L, E = itself
 * (Alg. 5).  Each iteration expands v = root.E (Alg. 2: all |A| Q-nodes; Alg. 3: n draws keyed as
 * in qvts_plan_step, one child per unique z, weight f/n, Eq. 3 posterior, Alg. 5 leaf bounds),
 * then updates v and its ancestors to the root: Alg. 6 with gamma (U_Q = R + gamma sum w U,
 * L_Q likewise; H_Q = gamma w H of the child maximising it; E_Q = its E), Alg. 7 (U = max U_Q,
 * L = max L_Q; H, E of the argmax-U_Q child).  Ties go to the lowest index.  planningFinished():
 * max_expansions reached, root U - L <= gap_tol, root.E at max_depth (terminal, H = 0), the node
 * pool full, or time_budget_ms (> 0) elapsed.  getOptimalAction(): max L_Q, ties by U_Q then
 * index; an unexpanded root takes the action of its PBVI arg-max vector.
 * Needs qvts_fib_iteration and qvts_pbvi.  root_dev: device fp32 [H*W].  Node beliefs stay in
 * HBM (H*W*4 bytes each); the pool holds 1 + max_expansions*|A|*min(n,16) V-nodes, capped at
 * half the free device memory.  Synchronises `stream` once or twice per expansion. */
typedef struct {
    int32_t n_samples;        /* draws per Q-node, 1..4096                                  */
    uint32_t seed, step, episode;
    int32_t sampler;          /* qvts_sampler                                               */
    int32_t max_expansions;   /* >= 0                                                       */
    int32_t max_depth;        /* 1..8                                                       */
    double gap_tol;           /* stop once root U - L <= gap_tol                            */
    double time_budget_ms;    /* > 0: also stop after this much wall-clock time (anytime)   */
    int32_t reuse;            /* 1: continue the kept tree (after qvts_bf_advance); root_dev
                                 is then ignored and may be NULL        */
} qvts_bf_cfg;
typedef enum { QVTS_BF_BUDGET = 0, QVTS_BF_GAP = 1, QVTS_BF_TERMINAL = 2, QVTS_BF_POOL = 3, QVTS_BF_TIME = 4 } qvts_bf_stop;
typedef struct {
    int32_t action;           /* stencil id                                                 */
    int32_t n_actions;
    int32_t n_expansions;
    int32_t stop_reason;      /* qvts_bf_stop                                               */
    int64_t n_vnodes;
    double U, L;              /* root bounds                                                */
    double u_q[9], l_q[9];    /* root Q-node bounds (NaN while the root is unexpanded)      */
    double device_ms;         /* CUDA-event time from the first to the last kernel          */
} qvts_bf_result;
QVTS_API qvts_status qvts_plan_best_first(qvts_model *model, const float *root_dev, const qvts_bf_cfg *cfg,
                                          qvts_bf_result *res, void *stream);
/* s.update(a, z) (Alg. 1, "set the root to be consistent with the current belief";
 * SPEC advance_root): if the root's Q-node for stencil id `action` has a child with observation z,
 * that V-node becomes the root and keeps its subtree: paths lose their first byte and depths drop
 * by one, so later draws are keyed relative to the new root; every other node is discarded
 * (depth -1 in the trace, pool slots not recycled).  *reused = 1 then, and the next
 * qvts_plan_best_first with cfg.reuse = 1 continues from it; *reused = 0 when z was not sampled
 * (or the root is unexpanded): build a fresh root from qvts_belief_update instead. */
QVTS_API qvts_status qvts_bf_advance(qvts_model *model, int32_t action, int32_t z, int32_t *reused, void *stream);
/* The last best-first tree (any pointer may be NULL): per V-node [n_v] path, depth (-1: discarded
 * by qvts_bf_advance), sampled count f, U, L, H, E (node index), expanded (0/1); exp_order
 * [n_expansions] = node indices expanded by the last call, in order; root_trace
 * [(n_expansions+1)][2] = root (U, L) before the first and after each expansion of that call. */
QVTS_API qvts_status qvts_trace_best_first(const qvts_model *model, int64_t *n_v, int32_t *n_expansions,
                                           uint64_t *path, int32_t *depth, int32_t *f, double *U, double *L,
                                           double *H, int32_t *E, int32_t *expanded, int32_t *exp_order,
                                           double *root_trace);

/* ---- (5) closed-loop episodes (Alg. 1 outer loop) -----
 * Each episode e draws x0 ~ b0 and then repeats: plan (QVTS over all active episodes at once,
 * or MDP on the belief mode), true motion y ~ T'(x,a,.) (an occupied/off-map y is a collision
 * and the robot stays), z ~ O(x',.), return += gamma^k R(x,a) (Eq. 1), b <- Phi(b,a,z) (Eq. 3),
 * until `stop_patience` consecutive stays (success iff at the goal) or max_steps (R26/R27).
 * Environment draws use Philox ctr = (0, 0, 0, step), key = (seed, episode): word 0 motion,
 * word 1 observation, word 2 the initial state (Appendix A.2).  Episodes with
 * e % nranks != rank are skipped when comm != NULL and their records reduced across ranks. */
/* Planners: QVTS; MDP = one Q table lookup at the belief mode; A* = unit-cost A* (reading R29)
 * from the belief mode, run on the host (the paper's two comparators). */
typedef enum { QVTS_PLANNER_QVTS = 0, QVTS_PLANNER_MDP = 1, QVTS_PLANNER_ASTAR = 2 } qvts_planner;
typedef struct {
    int32_t n_episodes, max_steps, stop_patience, planner, depth, n_samples;
    uint32_t seed;
    const float *b0_dev;          /* device fp32 [H*W]; NULL = uniform over free cells         */
    /* optional host logs [n_episodes][max_steps] (-1 after the episode ended): executed action
     * (stencil id), observation z, true state after the step.  NULL = not recorded. */
    int32_t *log_actions, *log_obs, *log_states;
} qvts_episode_cfg;
typedef struct {
    int32_t outcome;              /* 0 success, 1 wrong stop, 2 step cap, 3 zero likelihood    */
    int32_t steps, collisions, x0, x_final;
    double disc_return;
} qvts_episode_record;
QVTS_API qvts_status qvts_run_episodes(qvts_model *model, const qvts_episode_cfg *cfg, const qvts_comm *comm,
                              qvts_episode_record *out_host /*[n_episodes]*/, void *stream);

#ifdef __cplusplus
}
#endif
#endif /* QVTS_H */
