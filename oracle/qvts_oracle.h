/* qvts_oracle.h — TEST INFRASTRUCTURE ONLY.
 *
 * A plain, slow, fp64 CPU implementation of what the QVTS hot path computes, written from
 * the paper (arXiv 1810.00204, /root/reference/PAPER.md) and SURVEY.md §8(c).  Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline leg may load it.  It shares no code,
 * header, table or constant generator with the CUDA library under paper_1810_00204_b200/.
 *
 * Parity pins for every function are listed in DESIGN.md "Oracle pins"; the one function
 * without an independent pin is marked "parity unpinned" below.
 */
#ifndef QVTS_ORACLE_H
#define QVTS_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { OR_OK = 0, OR_ERR_INVALID_ARG = 1, OR_ERR_INVALID_MODEL = 2, OR_ERR_NOT_CONVERGED = 4,
       OR_ERR_ZERO_LIKELIHOOD = 5, OR_ERR_OUT_OF_MEMORY = 6 };

typedef struct or_model or_model;
typedef struct or_trace or_trace;

/* ---- model (PAPER.md:44 tuple; grid compile PAPER.md:305-355 §V) ---- */
or_model *or_grid_model_create(int H, int W, const uint8_t *occ, int goal, unsigned action_mask,
                               double p_int, double p_stay, double p_lat, double acc,
                               double gamma, int *status);
/* Generic dense model (T [nx][na][nx], O [nx][nz], R [nx][na]) for the SPEC Eq. 3 examples. */
or_model *or_dense_model_create(int nx, int na, int nz, const double *T, const double *O,
                                const double *R, double gamma, int *status);
void or_model_free(or_model *m);
int or_num_states(const or_model *m);
int or_num_actions(const or_model *m);
int or_num_obs(const or_model *m);
int or_action_id(const or_model *m, int a);          /* stencil id of action index a   */
double or_T(const or_model *m, int x, int a, int y);  /* clamped T(x,a,y) */
double or_Tprime(const or_model *m, int x, int a, int k); /* pre-clamp T'(x,a,N_k(x)), k=0..8 */
double or_O(const or_model *m, int x, int z);
double or_R(const or_model *m, int x, int a);
int or_sig(const or_model *m, int x);
int or_occ(const or_model *m, int x);

/* ---- RNG ---- */
void or_philox4x32_10(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]);
double or_uniform(uint32_t w);
/* A.5 inverse CDF over K weights; *flag set per A.6 (gap < 1e-6). */
int or_inverse_cdf(const double *p, int K, double u, int *flag);

/* ---- belief arithmetic (Eq. 3, R(b,a) PAPER.md:58) ---- */
void or_predict(const or_model *m, const double *b, int a, double *bbar);
void or_marginal(const or_model *m, const double *bbar, double *P);
double or_belief_reward(const or_model *m, const double *b, int a);
int or_belief_update(const or_model *m, const double *b, int a, int z, double *out, double *p_obs);

/* ---- MDP value iteration, Q layout [na][nx] ---- */
int or_value_iteration(const or_model *m, double eps, int max_sweeps, double *V, double *Q,
                       int *sweeps, double *resid);
/* Fast Informed Bound (Eq. 7): one alpha-vector per action, iterated from
 * alpha = R_max/(1-gamma) until max|alpha' - alpha| < eps; layout [na][nx].
 * Occupied grid cells: alpha = 0 (unreachable, as for Q). */
int or_fib(const or_model *m, double eps, int max_iter, double *alpha, int *iters, double *resid);
/* ---- PBVI lower bound (§IV-B) ----
 * Belief set: B0 = {b0}; each expansion round, for every point b (in order) and every action a
 * (ascending) one Alg. 4 sample (x ~ b, x' ~ T, z ~ O; Philox words 1..3 of counter
 * (a, point, round, 0x7BB1), key (seed, 0xB5E7)) gives the candidate Phi(b,a,z); the candidate
 * farthest in L1 from the set (as grown so far) is added if that distance is > 0 (ties: lowest a).
 * Backups: Gamma0 = {R_min/(1-gamma)}; a sweep replaces Gamma by one vector per point,
 * alpha_b = R(.,a*) + gamma sum_z g_{a*,z}^{alpha*_{a*,z}}, g_{a,z}^alpha(x) = sum_x' O(x',z)
 * T(x,a,x') alpha(x'), alpha*_{a,z} = argmax_{alpha in Gamma} b . g_{a,z}^alpha, a* = argmax_a of
 * b.R(.,a) + gamma sum_z max_alpha b . g (ties: lowest index). */
typedef struct or_pbvi or_pbvi;
or_pbvi *or_pbvi_build(const or_model *m, const double *b0, int expansions, int max_points, uint32_t seed,
                       int sweeps);
void or_pbvi_free(or_pbvi *p);
int or_pbvi_npoints(const or_pbvi *p);
int or_pbvi_nalpha(const or_pbvi *p);
void or_pbvi_point(const or_pbvi *p, int i, double *out);      /* belief point i [nx] */
void or_pbvi_alpha(const or_pbvi *p, int i, double *out, int *action);
double or_pbvi_value(const or_pbvi *p, const double *b);       /* V_PBVI(b) = max alpha . b */
/* Eq. 4 with alpha_a = Q(.,a): max_a sum_x b(x) Q(x,a); argmax lowest index. */
double or_qmdp_value(const or_model *m, const double *Q, const double *b, int *argmax);

/* ---- plan step (Alg. 1-7 read per SURVEY §8(c) O6) ---- */
enum { OR_MODE_FREQ = 0, OR_MODE_EXACT = 1, OR_MODE_BRUTE = 2 };
enum { OR_SAMPLER_MARGINAL = 0, OR_SAMPLER_ANCESTRAL = 1 };
typedef struct {
    int depth, n_samples, mode, threads;
    uint32_t seed, step, episode;
    int sampler;   /* OR_SAMPLER_MARGINAL (reading R9, Philox word 0) or OR_SAMPLER_ANCESTRAL
                      (Alg. 4 literal: x ~ b, x' ~ T(x,a,.), z ~ O(x',.) with words 1..3) */
    /* replay table for flagged, mismatched draws (SURVEY c.5 step 3): the GPU's observation
       z (marginal sampler) or its state index x (ancestral sampler; x' and z are then recomputed
       from that x) -- taken only when it borders the near CDF boundary */
    int n_replay;
    const uint64_t *replay_path;
    const int32_t *replay_j;
    const uint8_t *replay_z;
    const int32_t *replay_x;
} or_plan_cfg;

or_trace *or_trace_new(int capture_beliefs /*0 none, 1 all non-leaf V-nodes*/);
void or_trace_free(or_trace *t);
int64_t or_trace_nq(const or_trace *t);
int64_t or_trace_nv(const or_trace *t);
int32_t or_trace_nsamples(const or_trace *t);
/* Q-node records (n = or_trace_nq); P and cnt are [nq][16]; z/flag are [nq][n_samples]. */
void or_trace_export_q(const or_trace *t, uint64_t *path, int32_t *level, int32_t *action,
                       double *R, double *P, uint16_t *cnt, double *Q, uint8_t *z, uint8_t *flag);
/* V-node records (non-root); belief_idx = -1 when not captured. */
void or_trace_export_v(const or_trace *t, uint64_t *path, int32_t *level, double *V, int32_t *zobs,
                       int32_t *f, int64_t *belief_idx);
void or_trace_belief(const or_trace *t, int64_t belief_idx, double *out);

int or_plan(const or_model *m, const double *Q, const double *b0, const or_plan_cfg *cfg,
            int *action, double *qroot, or_trace *trace);
/* One Q-node's own step (predict, marginal, R, draws) without recursion. */
int or_qnode_sample(const or_model *m, const double *b, int a, uint64_t qpath, const or_plan_cfg *cfg,
                    double *P, double *R, uint8_t *z, uint8_t *flag, uint16_t *cnt);
/* Value of a V-node at `level` (root = 0) with the subtree below it, as in or_plan. */
double or_vnode_value(const or_model *m, const double *Q, const double *b, uint64_t vpath, int level,
                      const or_plan_cfg *cfg, double *qvals /*[na] or NULL*/);

/* ---- anytime best-first QVTS (Alg. 1-7 with U/L/H/E, Eq. 8) ----
 * Alg. 6 (with gamma, R13) on one Q-node from its children (ascending z): U_Q = R + gamma sum w U,
 * L_Q likewise; the heuristic child maximises gamma w H (ties lowest) and gives H_Q, E_Q. */
void or_bf_q_update(double R, double gamma, int nc, const double *w, const double *U, const double *L,
                    const double *H, const int *E, double *UQ, double *LQ, double *HQ, int *EQ);
/* Alg. 7 with the Sec. IV-C indicator read as "the argmax-U_Q child" (ties lowest). */
void or_bf_v_update(int na, const double *UQ, const double *LQ, const double *HQ, const int *EQ,
                    double *U, double *L, double *H, int *E);
typedef struct {
    int expansions;       /* budget: V-node expansions (Alg. 1 planningFinished)                 */
    int max_depth;        /* 1..8; leaves at this depth are terminal: H := 0 (reading B5)        */
    double gap_tol;       /* stop once root U - L <= gap_tol                       */
    int n_replay;         /* GPU expansion order (V-node paths); followed when admissible       */
    const uint64_t *replay_path;
    double replay_tol;    /* near-tie band of the admissibility check                            */
} or_bf_cfg;
typedef struct or_bf_tree or_bf_tree;
/* pcfg: n_samples, mode (FREQ: weights f/n; EXACT: every z with P > 0, weight P), seed, step,
 * episode, sampler.  alphaU [nU][nx] (FIB), alphaL [nL][nx] with actions actL (PBVI). */
or_bf_tree *or_bf_plan(const or_model *m, const double *alphaU, int nU, const double *alphaL, int nL,
                       const int *actL, const double *b0, const or_plan_cfg *pcfg, const or_bf_cfg *bcfg);
void or_bf_free(or_bf_tree *t);
/* More expansions from the current root (after or_bf_advance: tree reuse). */
int or_bf_continue(or_bf_tree *t, const double *alphaU, int nU, const double *alphaL, int nL, const int *actL,
                   const or_plan_cfg *pcfg, const or_bf_cfg *bcfg);
/* s.update(a, z) (Alg. 1): re-root at the root's (a, z) child if it was sampled (returns 1) and
 * discard the rest (depth -1); paths/depths become relative to the new root. */
int or_bf_advance(or_bf_tree *t, int a_id, int z);
int or_bf_root_index(const or_bf_tree *t);
void or_bf_belief(const or_bf_tree *t, int i, double *out);   /* V-node i's belief [nx] */
/* action (stencil id), stop reason (0 budget, 1 gap, 2 terminal leaf selected), expansions done,
 * V-nodes, replay substitutions (admissible GPU choices that differ) and mismatches. */
void or_bf_summary(const or_bf_tree *t, int *action, int *stop, int *n_exp, int *n_v, int *subs, int *mism);
void or_bf_root(const or_bf_tree *t, double *U, double *L, double *UQ, double *LQ);   /* UQ/LQ [na] or NULL */
void or_bf_vnode(const or_bf_tree *t, int i, uint64_t *path, int *depth, int *f, double *w, double *U,
                 double *L, double *H, int *E, int *expanded);
uint64_t or_bf_expanded(const or_bf_tree *t, int k);    /* path of the k-th expanded V-node   */
void or_bf_root_trace(const or_bf_tree *t, int k, double *U, double *L);   /* root U, L after k expansions */

/* ---- episodes (reading R26/R27) ---- */
enum { OR_PLANNER_QVTS = 0, OR_PLANNER_MDP = 1, OR_PLANNER_ASTAR = 2 };
typedef struct {
    int planner, depth, n_samples, max_steps, stop_patience;
    uint32_t seed, episode;
} or_episode_cfg;
typedef struct {
    int32_t outcome;   /* 0 success, 1 wrong-stop, 2 step cap, 3 model error */
    int32_t steps, collisions, x0, x_final;
    double disc_return;
} or_episode_record;
/* log_* arrays (optional, size max_steps): executed action id, observation, true state after. */
int or_run_episode(const or_model *m, const double *Q, const double *b0, const or_episode_cfg *cfg,
                   or_episode_record *rec, int32_t *log_a, int32_t *log_z, int32_t *log_x);
int or_astar_action(const or_model *m, int start);   /* first stencil id of an A* path */
int or_astar_length(const or_model *m, int start);   /* path length, -1 if unreachable */
int or_belief_mode(const or_model *m, const double *b);
int or_ancestral_sample(const or_model *m, const double *b, int a, const uint32_t ctr[4],
                        const uint32_t key[2]);       /* Alg. 4 literal, Philox words 1..3 */

#ifdef __cplusplus
}
#endif
#endif
