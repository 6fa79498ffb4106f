/* qvts_oracle.c — TEST INFRASTRUCTURE ONLY (see qvts_oracle.h).
 *
 * Plain fp64 C, scalar loops, recursive depth-first tree.  Every function cites the passage
 * of PAPER.md (arXiv 1810.00204) or the SURVEY.md reading it follows.  Nothing here is
 * blocked, fused or reordered beyond what the cited definition states.
 */
#include "qvts_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define OR_NZ_GRID 16
#define OR_ZERO_LIK 1e-300      /* SPEC.md:55, 96 (reading R25) */
#define OR_FLAG_GAP 1e-6        /* SURVEY A.6 / north star "CDF gap under 1e-6" (R11) */

struct or_model {
    int nx, na, nz;
    double gamma;
    /* sparse clamped T rows: row (x,a) = entries [t_start[x*na+a], t_start[x*na+a+1]) */
    int *t_start, *t_y;
    double *t_p;
    double *O;          /* [nx][nz] */
    double *R;          /* [nx][na] */
    /* grid-only data (is_grid = 1) */
    int is_grid, H, W, goal;
    int action_id[9];
    uint8_t *occ;       /* [nx] */
    int *sig;           /* [nx] */
    double *Tp;         /* pre-clamp T'(x,a,k): [nx][na][9] */
};

/* ------------------------------------------------------------------------------------------ */
/* Grid geometry ("N_4(x) = x").                        */
static int stencil_dr(int k) { return k / 3 - 1; }
static int stencil_dc(int k) { return k % 3 - 1; }

/* occ(y) = 1 if y is off-map or m(y) = 1 (reading R4). Returns the neighbour cell or -1. */
static int grid_neighbour(const or_model *m, int x, int k, int *occupied) {
    int r = x / m->W + stencil_dr(k), c = x % m->W + stencil_dc(k);
    if (r < 0 || r >= m->H || c < 0 || c >= m->W) { *occupied = 1; return -1; }
    int y = r * m->W + c;
    *occupied = m->occ[y] ? 1 : 0;
    return y;
}

/* Ring of the 8 moving actions, clockwise from up-left (reading R3). */
static const int RING[8] = {0, 1, 2, 5, 8, 7, 6, 3};

/* Pre-clamp T'(x,a,.) over stencil offsets k (Fig. 2 unreadable -> reading R1/R2). */
static void grid_tprime(int a_id, double p_int, double p_stay, double p_lat, double w[9]) {
    for (int k = 0; k < 9; ++k) w[k] = 0.0;
    if (a_id == 4) { w[4] = 1.0; return; }           /* stay is deterministic (R2) */
    int i = 0;
    while (RING[i] != a_id) ++i;
    w[a_id] += p_int;
    w[4] += p_stay;
    w[RING[(i + 7) % 8]] += p_lat;
    w[RING[(i + 1) % 8]] += p_lat;
}

static void model_free_arrays(or_model *m) {
    free(m->t_start); free(m->t_y); free(m->t_p); free(m->O); free(m->R);
    free(m->occ); free(m->sig); free(m->Tp);
}

void or_model_free(or_model *m) {
    if (!m) return;
    model_free_arrays(m);
    free(m);
}

or_model *or_grid_model_create(int H, int W, const uint8_t *occ, int goal, unsigned action_mask,
                               double p_int, double p_stay, double p_lat, double acc,
                               double gamma, int *status) {
    *status = OR_ERR_INVALID_MODEL;
    if (H <= 0 || W <= 0 || !occ) return NULL;
    if (goal < 0 || goal >= H * W || occ[goal]) return NULL;
    if (p_int < 0 || p_stay < 0 || p_lat < 0 || fabs(p_int + p_stay + 2 * p_lat - 1.0) > 1e-9)
        return NULL;
    if (!(acc > 0.5 && acc <= 1.0)) return NULL;
    if (!(gamma > 0.0 && gamma < 1.0)) return NULL;
    action_mask &= 0x1FF;
    if (!action_mask) return NULL;

    or_model *m = (or_model *)calloc(1, sizeof(or_model));
    m->is_grid = 1; m->H = H; m->W = W; m->goal = goal; m->gamma = gamma;
    m->nx = H * W; m->nz = OR_NZ_GRID;
    for (int k = 0; k < 9; ++k) if (action_mask & (1u << k)) m->action_id[m->na++] = k;
    int nx = m->nx, na = m->na;
    m->occ = (uint8_t *)malloc(nx);
    for (int x = 0; x < nx; ++x) m->occ[x] = occ[x] ? 1 : 0;

    /* Signature: bit k <-> sensor N_{2k+1} (reading R6; PAPER.md:336 sensors N1,N3,N5,N7). */
    m->sig = (int *)malloc(sizeof(int) * nx);
    for (int x = 0; x < nx; ++x) {
        int s = 0, o;
        for (int k = 0; k < 4; ++k) { grid_neighbour(m, x, 2 * k + 1, &o); s |= o << k; }
        m->sig[x] = s;
    }
    /* O(x,z) = prod over 4 independent sensors, each correct w.p. acc (R7);
     * occupied x: uniform (reading R5). */
    m->O = (double *)malloc(sizeof(double) * nx * m->nz);
    for (int x = 0; x < nx; ++x)
        for (int z = 0; z < m->nz; ++z) {
            double o = 1.0;
            if (m->occ[x]) o = 1.0 / 16.0;
            else
                for (int k = 0; k < 4; ++k)
                    o *= (((z >> k) & 1) == ((m->sig[x] >> k) & 1)) ? acc : (1.0 - acc);
            m->O[x * m->nz + z] = o;
        }
    /* T' and clamped T (mass on occupied y is accumulated to x). */
    m->Tp = (double *)calloc((size_t)nx * na * 9, sizeof(double));
    m->t_start = (int *)malloc(sizeof(int) * (nx * na + 1));
    m->t_y = (int *)malloc(sizeof(int) * nx * na * 9);
    m->t_p = (double *)malloc(sizeof(double) * nx * na * 9);
    int ne = 0;
    for (int x = 0; x < nx; ++x)
        for (int a = 0; a < na; ++a) {
            double w[9];
            grid_tprime(m->action_id[a], p_int, p_stay, p_lat, w);
            memcpy(&m->Tp[((size_t)x * na + a) * 9], w, sizeof(w));
            m->t_start[x * na + a] = ne;
            if (m->occ[x]) {                       /* absorbing occupied rows (R5) */
                m->t_y[ne] = x; m->t_p[ne] = 1.0; ++ne;
                continue;
            }
            int row0 = ne;
            for (int k = 0; k < 9; ++k) {
                if (w[k] == 0.0) continue;
                int o, y = grid_neighbour(m, x, k, &o);
                if (k == 4) { y = x; o = 0; }
                if (o) y = x;                       /* clamp */
                int found = -1;
                for (int e = row0; e < ne; ++e) if (m->t_y[e] == y) found = e;
                if (found >= 0) m->t_p[found] += w[k];
                else { m->t_y[ne] = y; m->t_p[ne] = w[k]; ++ne; }
            }
        }
    m->t_start[nx * na] = ne;
    /* Reward: r(y) in {-2,-1,0}; R(x,4) = -2 off-goal; otherwise
     * R(x,a) = sum_y r(y) T'(x,a,y) with the PRE-clamp T', off-map y counted as occupied (R22). */
    m->R = (double *)malloc(sizeof(double) * nx * na);
    for (int x = 0; x < nx; ++x)
        for (int a = 0; a < na; ++a) {
            double v = 0.0;
            if (m->occ[x]) v = 0.0;                 /* unused (R5) */
            else if (m->action_id[a] == 4 && x != goal) v = -2.0;
            else {
                const double *w = &m->Tp[((size_t)x * na + a) * 9];
                for (int k = 0; k < 9; ++k) {
                    if (w[k] == 0.0) continue;
                    int o, y = grid_neighbour(m, x, k, &o);
                    if (k == 4) { y = x; o = 0; }
                    double r = o ? -2.0 : (y == goal ? 0.0 : -1.0);
                    v += r * w[k];
                }
            }
            m->R[x * na + a] = v;
        }
    *status = OR_OK;
    return m;
}

or_model *or_dense_model_create(int nx, int na, int nz, const double *T, const double *O,
                                const double *R, double gamma, int *status) {
    *status = OR_ERR_INVALID_MODEL;
    if (nx <= 0 || na <= 0 || nz <= 0 || !(gamma > 0 && gamma < 1)) return NULL;
    or_model *m = (or_model *)calloc(1, sizeof(or_model));
    m->nx = nx; m->na = na; m->nz = nz; m->gamma = gamma;
    for (int a = 0; a < na && a < 9; ++a) m->action_id[a] = a;
    m->t_start = (int *)malloc(sizeof(int) * (nx * na + 1));
    m->t_y = (int *)malloc(sizeof(int) * (size_t)nx * na * nx);
    m->t_p = (double *)malloc(sizeof(double) * (size_t)nx * na * nx);
    int ne = 0;
    for (int x = 0; x < nx; ++x)
        for (int a = 0; a < na; ++a) {
            m->t_start[x * na + a] = ne;
            double s = 0;
            for (int y = 0; y < nx; ++y) {
                double p = T[((size_t)x * na + a) * nx + y];
                if (p < 0) { or_model_free(m); return NULL; }
                s += p;
                if (p > 0) { m->t_y[ne] = y; m->t_p[ne] = p; ++ne; }
            }
            if (fabs(s - 1.0) > 1e-9) { or_model_free(m); return NULL; }
        }
    m->t_start[nx * na] = ne;
    m->O = (double *)malloc(sizeof(double) * nx * nz);
    memcpy(m->O, O, sizeof(double) * nx * nz);
    m->R = (double *)malloc(sizeof(double) * nx * na);
    memcpy(m->R, R, sizeof(double) * nx * na);
    *status = OR_OK;
    return m;
}

int or_num_states(const or_model *m) { return m->nx; }
int or_num_actions(const or_model *m) { return m->na; }
int or_num_obs(const or_model *m) { return m->nz; }
int or_action_id(const or_model *m, int a) { return m->action_id[a]; }
double or_O(const or_model *m, int x, int z) { return m->O[x * m->nz + z]; }
double or_R(const or_model *m, int x, int a) { return m->R[x * m->na + a]; }
int or_sig(const or_model *m, int x) { return m->is_grid ? m->sig[x] : 0; }
int or_occ(const or_model *m, int x) { return m->is_grid ? m->occ[x] : 0; }
double or_T(const or_model *m, int x, int a, int y) {
    double p = 0.0;
    for (int e = m->t_start[x * m->na + a]; e < m->t_start[x * m->na + a + 1]; ++e)
        if (m->t_y[e] == y) p += m->t_p[e];
    return p;
}
double or_Tprime(const or_model *m, int x, int a, int k) {
    return m->is_grid ? m->Tp[((size_t)x * m->na + a) * 9 + k] : 0.0;
}

/* ------------------------------------------------------------------------------------------ */
/* Philox4x32-10 (Salmon et al. 2011).                                   */
void or_philox4x32_10(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]) {
    uint32_t c0 = ctr[0], c1 = ctr[1], c2 = ctr[2], c3 = ctr[3];
    uint32_t k0 = key[0], k1 = key[1];
    for (int round = 0; round < 10; ++round) {
        if (round > 0) { k0 += 0x9E3779B9u; k1 += 0xBB67AE85u; }
        uint64_t p0 = (uint64_t)0xD2511F53u * c0;
        uint64_t p1 = (uint64_t)0xCD9E8D57u * c2;
        uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
        uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
        uint32_t n0 = hi1 ^ c1 ^ k0, n1 = lo1, n2 = hi0 ^ c3 ^ k1, n3 = lo0;
        c0 = n0; c1 = n1; c2 = n2; c3 = n3;
    }
    out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

/* A.4: u = ((w >> 8) + 0.5) * 2^-24 */
double or_uniform(uint32_t w) { return ((double)(w >> 8) + 0.5) * (1.0 / 16777216.0); }

/* A.5: C_k = sum_{i<=k} p_i ascending in fp64; result = min{k : u*C_{K-1} < C_k}.
 * A.6: flag when min_{k<K-1} |u*C_{K-1} - C_k| < 1e-6. */
int or_inverse_cdf(const double *p, int K, double u, int *flag) {
    double *C = (double *)malloc(sizeof(double) * K);
    double s = 0.0;
    for (int k = 0; k < K; ++k) { s += p[k]; C[k] = s; }
    double t = u * C[K - 1];
    int res = K - 1;
    for (int k = 0; k < K; ++k) if (t < C[k]) { res = k; break; }
    if (flag) {
        *flag = 0;
        for (int k = 0; k < K - 1; ++k) if (fabs(t - C[k]) < OR_FLAG_GAP) *flag = 1;
    }
    free(C);
    return res;
}

/* ------------------------------------------------------------------------------------------ */
/* Eq. 3 inner sum, scatter form: bbar(y) = sum_x T(x,a,y) b(x).          */
void or_predict(const or_model *m, const double *b, int a, double *bbar) {
    for (int y = 0; y < m->nx; ++y) bbar[y] = 0.0;
    for (int x = 0; x < m->nx; ++x) {
        if (b[x] == 0.0) continue;
        for (int e = m->t_start[x * m->na + a]; e < m->t_start[x * m->na + a + 1]; ++e)
            bbar[m->t_y[e]] += m->t_p[e] * b[x];
    }
}

/* Normaliser of Eq. 3: P(z|b,a) = sum_y O(y,z) bbar(y). */
void or_marginal(const or_model *m, const double *bbar, double *P) {
    for (int z = 0; z < m->nz; ++z) {
        double s = 0.0;
        for (int y = 0; y < m->nx; ++y) s += m->O[y * m->nz + z] * bbar[y];
        P[z] = s;
    }
}

/* R(b,a) = sum_x R(x,a) b(x). */
double or_belief_reward(const or_model *m, const double *b, int a) {
    double s = 0.0;
    for (int x = 0; x < m->nx; ++x) s += m->R[x * m->na + a] * b[x];
    return s;
}

/* Eq. 3: Phi(b,a,z)(x') = O(x',z) sum_x T(x,a,x') b(x) / P(z|b,a). */
int or_belief_update(const or_model *m, const double *b, int a, int z, double *out, double *p_obs) {
    if (a < 0 || a >= m->na || z < 0 || z >= m->nz) return OR_ERR_INVALID_ARG;
    double *bbar = (double *)malloc(sizeof(double) * m->nx);
    double *P = (double *)malloc(sizeof(double) * m->nz);
    or_predict(m, b, a, bbar);
    or_marginal(m, bbar, P);
    double pz = P[z];
    if (p_obs) *p_obs = pz;
    int st = OR_OK;
    if (pz <= OR_ZERO_LIK) st = OR_ERR_ZERO_LIKELIHOOD;
    else
        for (int y = 0; y < m->nx; ++y) out[y] = m->O[y * m->nz + z] * bbar[y] / pz;
    free(bbar); free(P);
    return st;
}

/* ------------------------------------------------------------------------------------------ */
/* MDP value iteration ("self-implemented value iteration"; reading R24):
 * synchronous Jacobi from V0 = 0, Q_k(x,a) = R(x,a) + gamma sum_y T(x,a,y) V_k(y),
 * V_{k+1} = max_a Q_k, stop when max|V_{k+1} - V_k| < eps; then Q = R + gamma T V.
 * Occupied grid cells: V = Q = 0 (reading R5). */
static double bellman_q(const or_model *m, const double *V, int x, int a) {
    double s = 0.0;
    for (int e = m->t_start[x * m->na + a]; e < m->t_start[x * m->na + a + 1]; ++e)
        s += m->t_p[e] * V[m->t_y[e]];
    return m->R[x * m->na + a] + m->gamma * s;
}

int or_value_iteration(const or_model *m, double eps, int max_sweeps, double *V, double *Q,
                       int *sweeps, double *resid) {
    int nx = m->nx, na = m->na;
    double *Vn = (double *)malloc(sizeof(double) * nx);
    for (int x = 0; x < nx; ++x) V[x] = 0.0;
    int k = 0, st = OR_ERR_NOT_CONVERGED;
    double res = INFINITY;
    while (k < max_sweeps) {
        res = 0.0;
        for (int x = 0; x < nx; ++x) {
            if (m->is_grid && m->occ[x]) { Vn[x] = 0.0; continue; }
            double best = -INFINITY;
            for (int a = 0; a < na; ++a) {
                double q = bellman_q(m, V, x, a);
                if (q > best) best = q;
            }
            Vn[x] = best;
            double d = fabs(best - V[x]);
            if (d > res) res = d;
        }
        memcpy(V, Vn, sizeof(double) * nx);
        ++k;
        if (res < eps) { st = OR_OK; break; }
    }
    for (int a = 0; a < na; ++a)
        for (int x = 0; x < nx; ++x)
            Q[(size_t)a * nx + x] = (m->is_grid && m->occ[x]) ? 0.0 : bellman_q(m, V, x, a);
    if (sweeps) *sweeps = k;
    if (resid) *resid = res;
    free(Vn);
    return st;
}

/* Fast Informed Bound, Eq. 7:
 *   alpha^a(x) = R(x,a) + gamma sum_z max_a' sum_x' O(x',z) T(x,a,x') alpha^a'(x'),
 * a monotone contraction; synchronous iteration from alpha = R_max/(1-gamma). */
int or_fib(const or_model *m, double eps, int max_iter, double *alpha, int *iters, double *resid) {
    int nx = m->nx, na = m->na, nz = m->nz;
    double rmax = -INFINITY;   /* over reachable states: occupied grid rows carry R := 0 (R5) */
    for (int i = 0; i < nx * na; ++i)
        if (!(m->is_grid && m->occ[i / na]) && m->R[i] > rmax) rmax = m->R[i];
    double *an = (double *)malloc(sizeof(double) * (size_t)na * nx);
    for (int a = 0; a < na; ++a)
        for (int x = 0; x < nx; ++x)
            alpha[(size_t)a * nx + x] = (m->is_grid && m->occ[x]) ? 0.0 : rmax / (1.0 - m->gamma);
    int k = 0, st = OR_ERR_NOT_CONVERGED;
    double res = INFINITY;
    while (k < max_iter) {
        res = 0.0;
        for (int x = 0; x < nx; ++x)
            for (int a = 0; a < na; ++a) {
                double v = 0.0;
                if (!(m->is_grid && m->occ[x])) {
                    double s = 0.0;
                    for (int z = 0; z < nz; ++z) {
                        double best = -INFINITY;
                        for (int a2 = 0; a2 < na; ++a2) {
                            double d = 0.0;
                            for (int e = m->t_start[x * na + a]; e < m->t_start[x * na + a + 1]; ++e) {
                                int y = m->t_y[e];
                                d += m->O[y * nz + z] * m->t_p[e] * alpha[(size_t)a2 * nx + y];
                            }
                            if (d > best) best = d;
                        }
                        s += best;
                    }
                    v = m->R[x * na + a] + m->gamma * s;
                }
                an[(size_t)a * nx + x] = v;
                double dd = fabs(v - alpha[(size_t)a * nx + x]);
                if (dd > res) res = dd;
            }
        memcpy(alpha, an, sizeof(double) * (size_t)na * nx);
        ++k;
        if (res < eps) { st = OR_OK; break; }
    }
    if (iters) *iters = k;
    if (resid) *resid = res;
    free(an);
    return st;
}

/* ---- PBVI (§IV-B) ------------------------------------------------------------------------------ */
static int ancestral_draw(const or_model *m, const double *b, int a, const uint32_t w[4], int *flag);
/* PBVI arg-max rule (reading B4): v replaces the incumbent only if it is larger by more
 * than 1e-10 (1 + |incumbent|) -> near-ties go to the lowest index on any summation order. */
#define OR_PBVI_TIE 1e-10
static int pbvi_beats(double v, double best) { return v > best + OR_PBVI_TIE * (1.0 + fabs(best)); }
struct or_pbvi {
    int nx, nb, na_alpha;
    double *B;        /* [nb][nx] */
    double *G;        /* [na_alpha][nx] */
    int *gact;
};

/* b . g_{a,z}^alpha = sum_x b(x) sum_x' O(x',z) T(x,a,x') alpha(x') (scatter over T rows) */
static double pbvi_dot(const or_model *m, const double *b, int a, int z, const double *alpha) {
    double s = 0.0;
    for (int x = 0; x < m->nx; ++x) {
        if (b[x] == 0.0) continue;
        double g = 0.0;
        for (int e = m->t_start[x * m->na + a]; e < m->t_start[x * m->na + a + 1]; ++e) {
            int y = m->t_y[e];
            g += m->O[y * m->nz + z] * m->t_p[e] * alpha[y];
        }
        s += b[x] * g;
    }
    return s;
}

or_pbvi *or_pbvi_build(const or_model *m, const double *b0, int expansions, int max_points, uint32_t seed,
                       int sweeps) {
    int nx = m->nx, na = m->na, nz = m->nz;
    or_pbvi *p = (or_pbvi *)calloc(1, sizeof(or_pbvi));
    p->nx = nx;
    p->B = (double *)malloc(sizeof(double) * nx * (size_t)(max_points > 0 ? max_points : 1));
    memcpy(p->B, b0, sizeof(double) * nx);
    p->nb = 1;
    double *cand = (double *)malloc(sizeof(double) * nx * na);
    /* belief set expansion */
    for (int r = 0; r < expansions && p->nb < max_points; ++r) {
        int n0 = p->nb;
        for (int i = 0; i < n0 && p->nb < max_points; ++i) {
            const double *b = &p->B[(size_t)i * nx];
            int best_a = -1;
            double best_d = 0.0;
            for (int a = 0; a < na; ++a) {
                uint32_t ctr[4] = {(uint32_t)a, (uint32_t)i, (uint32_t)r, 0x7BB1u}, key[2] = {seed, 0xB5E7u}, w[4];
                or_philox4x32_10(ctr, key, w);
                int z = ancestral_draw(m, b, a, w, NULL);
                double pz;
                if (or_belief_update(m, b, a, z, &cand[(size_t)a * nx], &pz) != OR_OK) continue;
                double dmin = INFINITY;      /* L1 distance to the set as grown so far */
                for (int k = 0; k < p->nb; ++k) {
                    double d = 0.0;
                    for (int x = 0; x < nx; ++x) d += fabs(cand[(size_t)a * nx + x] - p->B[(size_t)k * nx + x]);
                    if (d < dmin) dmin = d;
                }
                if (pbvi_beats(dmin, best_d)) { best_d = dmin; best_a = a; }
            }
            if (best_a >= 0) {
                memcpy(&p->B[(size_t)p->nb * nx], &cand[(size_t)best_a * nx], sizeof(double) * nx);
                p->nb++;
            }
        }
    }
    free(cand);
    /* point-based backups from the blind lower bound */
    double rmin = INFINITY;
    for (int i = 0; i < nx * na; ++i)
        if (!(m->is_grid && m->occ[i / na]) && m->R[i] < rmin) rmin = m->R[i];
    p->na_alpha = 1;
    p->G = (double *)malloc(sizeof(double) * nx * (size_t)(p->nb > 1 ? p->nb : 1));
    p->gact = (int *)calloc(p->nb > 1 ? p->nb : 1, sizeof(int));
    for (int x = 0; x < nx; ++x) p->G[x] = (m->is_grid && m->occ[x]) ? 0.0 : rmin / (1.0 - m->gamma);
    double *Gn = (double *)malloc(sizeof(double) * nx * (size_t)p->nb);
    int *an = (int *)malloc(sizeof(int) * p->nb);
    int *sel = (int *)malloc(sizeof(int) * na * nz);
    for (int sw = 0; sw < sweeps; ++sw) {
        for (int i = 0; i < p->nb; ++i) {
            const double *b = &p->B[(size_t)i * nx];
            double best_v = -INFINITY;
            int best_a = 0;
            for (int a = 0; a < na; ++a) {
                double v = or_belief_reward(m, b, a);
                double acc = 0.0;
                for (int z = 0; z < nz; ++z) {
                    double bz = 0.0;
                    int bk = 0;
                    for (int k = 0; k < p->na_alpha; ++k) {
                        double d = pbvi_dot(m, b, a, z, &p->G[(size_t)k * nx]);
                        if (k == 0 || pbvi_beats(d, bz)) { bz = d; bk = k; }
                    }
                    sel[a * nz + z] = bk;
                    acc += bz;
                }
                v += m->gamma * acc;
                if (a == 0 || pbvi_beats(v, best_v)) { best_v = v; best_a = a; }
            }
            /* alpha_b(x) = R(x,a*) + gamma sum_z sum_x' O(x',z) T(x,a*,x') alpha*_z(x') */
            double *out = &Gn[(size_t)i * nx];
            for (int x = 0; x < nx; ++x) {
                if (m->is_grid && m->occ[x]) { out[x] = 0.0; continue; }
                double acc = 0.0;
                for (int z = 0; z < nz; ++z) {
                    const double *al = &p->G[(size_t)sel[best_a * nz + z] * nx];
                    double g = 0.0;
                    for (int e = m->t_start[x * na + best_a]; e < m->t_start[x * na + best_a + 1]; ++e)
                        g += m->O[m->t_y[e] * nz + z] * m->t_p[e] * al[m->t_y[e]];
                    acc += g;
                }
                out[x] = m->R[x * na + best_a] + m->gamma * acc;
            }
            an[i] = m->action_id[best_a];
        }
        memcpy(p->G, Gn, sizeof(double) * nx * (size_t)p->nb);
        memcpy(p->gact, an, sizeof(int) * p->nb);
        p->na_alpha = p->nb;
    }
    free(Gn); free(an); free(sel);
    return p;
}
void or_pbvi_free(or_pbvi *p) {
    if (!p) return;
    free(p->B); free(p->G); free(p->gact); free(p);
}
int or_pbvi_npoints(const or_pbvi *p) { return p->nb; }
int or_pbvi_nalpha(const or_pbvi *p) { return p->na_alpha; }
void or_pbvi_point(const or_pbvi *p, int i, double *out) { memcpy(out, &p->B[(size_t)i * p->nx], sizeof(double) * p->nx); }
void or_pbvi_alpha(const or_pbvi *p, int i, double *out, int *action) {
    memcpy(out, &p->G[(size_t)i * p->nx], sizeof(double) * p->nx);
    if (action) *action = p->gact[i];
}
double or_pbvi_value(const or_pbvi *p, const double *b) {
    double best = -INFINITY;
    for (int k = 0; k < p->na_alpha; ++k) {
        double s = 0.0;
        for (int x = 0; x < p->nx; ++x) s += p->G[(size_t)k * p->nx + x] * b[x];
        if (s > best) best = s;
    }
    return best;
}

/* Eq. 4 with one alpha-vector per action, alpha_a = Q(.,a) (north star Q_MDP leaf; R14). */
double or_qmdp_value(const or_model *m, const double *Q, const double *b, int *argmax) {
    double best = -INFINITY;
    int arg = 0;
    for (int a = 0; a < m->na; ++a) {
        double s = 0.0;
        for (int x = 0; x < m->nx; ++x) s += b[x] * Q[(size_t)a * m->nx + x];
        if (s > best) { best = s; arg = a; }            /* ties -> lowest index (R16) */
    }
    if (argmax) *argmax = arg;
    return best;
}

/* ------------------------------------------------------------------------------------------ */
/* Trace storage.                                                                             */
typedef struct { uint64_t path; int32_t level, action; double R, Q; double P[16]; uint16_t cnt[16]; } qrec_t;
typedef struct { uint64_t path; int32_t level, z, f; double V; int64_t bidx; } vrec_t;

struct or_trace {
    int capture, n;
    int64_t nq, capq, nv, capv, nb, capb, nx;
    qrec_t *q; vrec_t *v;
    uint8_t *z, *flag;           /* [capq][n] */
    double *bel;                 /* [capb][nx] */
};

or_trace *or_trace_new(int capture_beliefs) {
    or_trace *t = (or_trace *)calloc(1, sizeof(or_trace));
    t->capture = capture_beliefs;
    return t;
}
void or_trace_free(or_trace *t) {
    if (!t) return;
    free(t->q); free(t->v); free(t->z); free(t->flag); free(t->bel); free(t);
}
int64_t or_trace_nq(const or_trace *t) { return t->nq; }
int64_t or_trace_nv(const or_trace *t) { return t->nv; }
int32_t or_trace_nsamples(const or_trace *t) { return t->n; }

static int64_t trace_add_q(or_trace *t, int n) {
    if (t->nq == t->capq) {
        t->capq = t->capq ? 2 * t->capq : 64;
        t->q = (qrec_t *)realloc(t->q, sizeof(qrec_t) * t->capq);
        t->z = (uint8_t *)realloc(t->z, (size_t)t->capq * (n > 0 ? n : 1));
        t->flag = (uint8_t *)realloc(t->flag, (size_t)t->capq * (n > 0 ? n : 1));
    }
    return t->nq++;
}
static int64_t trace_add_v(or_trace *t) {
    if (t->nv == t->capv) {
        t->capv = t->capv ? 2 * t->capv : 64;
        t->v = (vrec_t *)realloc(t->v, sizeof(vrec_t) * t->capv);
    }
    return t->nv++;
}
static int64_t trace_add_belief(or_trace *t, const double *b) {
    if (t->nb == t->capb) {
        t->capb = t->capb ? 2 * t->capb : 16;
        t->bel = (double *)realloc(t->bel, sizeof(double) * t->capb * t->nx);
    }
    memcpy(&t->bel[t->nb * t->nx], b, sizeof(double) * t->nx);
    return t->nb++;
}

void or_trace_export_q(const or_trace *t, uint64_t *path, int32_t *level, int32_t *action,
                       double *R, double *P, uint16_t *cnt, double *Q, uint8_t *z, uint8_t *flag) {
    for (int64_t i = 0; i < t->nq; ++i) {
        path[i] = t->q[i].path; level[i] = t->q[i].level; action[i] = t->q[i].action;
        R[i] = t->q[i].R; Q[i] = t->q[i].Q;
        for (int k = 0; k < 16; ++k) { P[i * 16 + k] = t->q[i].P[k]; cnt[i * 16 + k] = t->q[i].cnt[k]; }
    }
    if (t->n > 0) {
        memcpy(z, t->z, (size_t)t->nq * t->n);
        memcpy(flag, t->flag, (size_t)t->nq * t->n);
    }
}
void or_trace_export_v(const or_trace *t, uint64_t *path, int32_t *level, double *V, int32_t *zobs,
                       int32_t *f, int64_t *belief_idx) {
    for (int64_t i = 0; i < t->nv; ++i) {
        path[i] = t->v[i].path; level[i] = t->v[i].level; V[i] = t->v[i].V;
        zobs[i] = t->v[i].z; f[i] = t->v[i].f; belief_idx[i] = t->v[i].bidx;
    }
}
void or_trace_belief(const or_trace *t, int64_t bi, double *out) {
    memcpy(out, &t->bel[bi * t->nx], sizeof(double) * t->nx);
}

/* ------------------------------------------------------------------------------------------ */
/* Plan step: SURVEY §8(c) O6.  Alg. 2 creates all |A| Q-nodes of a V-node;
 * Alg. 3 draws n observations (Alg. 4 distribution, reading R9, keyed by
 * tree path per Appendix A), keeps the unique ones with their frequency as weight
 * (R12), builds one child per unique z with Eq. 3, and updates q
 * (Alg. 6 with gamma, reading R13); Alg. 7 takes V = max_a Q.  Leaves use Q_MDP (R14).     */
typedef struct {
    const or_model *m;
    const double *Q;
    const or_plan_cfg *cfg;
    or_trace *tr;
} plan_ctx;

static uint64_t qpath_of(uint64_t vpath, int level, int a_id) {
    return vpath | ((uint64_t)(a_id + 1) << (8 * level));
}
static uint64_t vpath_of(uint64_t qpath, int level, int z) {
    return qpath | ((uint64_t)z << (8 * level + 4));
}

static int replay_lookup(const or_plan_cfg *cfg, uint64_t qpath, int j, int *z) {
    for (int i = 0; i < cfg->n_replay; ++i)
        if (cfg->replay_path[i] == qpath && cfg->replay_j[i] == j) { *z = cfg->replay_z[i]; return 1; }
    return 0;
}
static int replay_lookup_x(const or_plan_cfg *cfg, uint64_t qpath, int j, int *x) {
    if (!cfg->replay_x) return 0;
    for (int i = 0; i < cfg->n_replay; ++i)
        if (cfg->replay_path[i] == qpath && cfg->replay_j[i] == j) { *x = cfg->replay_x[i]; return 1; }
    return 0;
}

/* c.5 step 3: a replayed category r of the inverse CDF over p[0..K) (target t = u * C_last) is
 * admissible only if it borders a boundary C_k within OR_FLAG_GAP of t: r is the first category
 * whose cumulative reaches C_k, or the first whose cumulative exceeds it. */
static int borders_near_boundary(const double *p, int K, double u, int r) {
    double *C = (double *)malloc(sizeof(double) * K);
    double s = 0.0;
    for (int k = 0; k < K; ++k) { s += p[k]; C[k] = s; }
    double t = u * C[K - 1];
    int ok = 0;
    for (int k = 0; k < K - 1 && !ok; ++k) {
        if (fabs(t - C[k]) >= OR_FLAG_GAP) continue;
        int lo = K - 1, hi = K - 1;
        for (int i = 0; i < K; ++i) if (C[i] >= C[k]) { lo = i; break; }
        for (int i = 0; i < K; ++i) if (C[i] > C[k]) { hi = i; break; }
        ok = (r == lo || r == hi);
    }
    free(C);
    return ok;
}

/* Draws of one Q-node (Appendix A.2-A.6); returns the draws, flags and counts. */
/* Alg. 4 literal: x ~ b (word 1), x' ~ T(x,a,.) over the clamped row in its
 * stored order (word 2), z ~ O(x',.) (word 3).  Only the state draw can be near a CDF boundary
 * (the other two CDFs are exact model tables), so the flag reports that draw (A.6 rule). */
static int ancestral_state(const or_model *m, const double *b, const uint32_t w[4], int *flag) {
    return or_inverse_cdf(b, m->nx, or_uniform(w[1]), flag);
}
static int ancestral_obs(const or_model *m, int x, int a, const uint32_t w[4]) {
    int e0 = m->t_start[x * m->na + a], e1 = m->t_start[x * m->na + a + 1];
    double p[9];
    for (int e = e0; e < e1; ++e) p[e - e0] = m->t_p[e];
    int xp = m->t_y[e0 + or_inverse_cdf(p, e1 - e0, or_uniform(w[2]), NULL)];
    return or_inverse_cdf(&m->O[xp * m->nz], m->nz, or_uniform(w[3]), NULL);
}
static int ancestral_draw(const or_model *m, const double *b, int a, const uint32_t w[4], int *flag) {
    return ancestral_obs(m, ancestral_state(m, b, w, flag), a, w);
}

static void qnode_draws(const or_model *m, const double *b, int a, const or_plan_cfg *cfg, int nz,
                        const double *P, uint64_t qpath, uint8_t *zs, uint8_t *flags, uint16_t *cnt) {
    for (int k = 0; k < nz; ++k) cnt[k] = 0;
    for (int j = 0; j < cfg->n_samples; ++j) {
        uint32_t ctr[4] = {(uint32_t)j, (uint32_t)qpath, (uint32_t)(qpath >> 32), cfg->step};
        uint32_t key[2] = {cfg->seed, cfg->episode}, w[4];
        or_philox4x32_10(ctr, key, w);
        if (cfg->sampler == OR_SAMPLER_ANCESTRAL) {
            int flag, xr;
            int x = ancestral_state(m, b, w, &flag);
            /* a flagged state draw may land in the neighbouring state: take the GPU's x if it
               borders the near boundary, then x' and z follow from it with words 2-3 */
            if (flag && cfg->n_replay > 0 && replay_lookup_x(cfg, qpath, j, &xr) && xr != x &&
                xr >= 0 && xr < m->nx && borders_near_boundary(b, m->nx, or_uniform(w[1]), xr))
                x = xr;
            int z = ancestral_obs(m, x, a, w);
            zs[j] = (uint8_t)z;
            flags[j] = (uint8_t)flag;
            cnt[z]++;
            continue;
        }
        double u = or_uniform(w[0]);
        int flag;
        int z = or_inverse_cdf(P, nz, u, &flag);
        int zr;
        if (flag && cfg->n_replay > 0 && replay_lookup(cfg, qpath, j, &zr) && zr != z &&
            borders_near_boundary(P, nz, u, zr))   /* accept only a category bordering a near boundary */
            z = zr;
        zs[j] = (uint8_t)z;
        flags[j] = (uint8_t)flag;
        cnt[z]++;
    }
}

static double vnode_rec(plan_ctx *c, const double *b, uint64_t vpath, int level, double *qvals);

/* Q-node at `level` (its parent V-node is at `level`), with levels_left = depth - level. */
static double qnode_rec(plan_ctx *c, const double *b, int a, uint64_t qpath, int level) {
    const or_model *m = c->m;
    const or_plan_cfg *cfg = c->cfg;
    int nx = m->nx, nz = m->nz, n = cfg->n_samples;
    double *bbar = (double *)malloc(sizeof(double) * nx);
    double *child = (double *)malloc(sizeof(double) * nx);
    double P[16];
    uint16_t cnt[16];
    uint8_t *zs = (uint8_t *)calloc(n > 0 ? n : 1, 1), *flags = (uint8_t *)calloc(n > 0 ? n : 1, 1);
    or_predict(m, b, a, bbar);                            /* Eq. 3 inner sum */
    or_marginal(m, bbar, P);                              /* P(z|b,a)       */
    double R = or_belief_reward(m, b, a);                 /* R(b,a)         */
    if (cfg->mode == OR_MODE_BRUTE) { for (int z = 0; z < nz; ++z) cnt[z] = 0; }
    else qnode_draws(m, b, a, cfg, nz, P, qpath, zs, flags, cnt);  /* Alg. 3 l.4-5 */
    double acc = 0.0;
    for (int z = 0; z < nz; ++z) {                        /* unique z ascending (R17) */
        int take = (cfg->mode == OR_MODE_BRUTE) ? (P[z] > OR_ZERO_LIK) : (cnt[z] > 0);
        if (!take) continue;
        double w = (cfg->mode == OR_MODE_FREQ) ? (double)cnt[z] / (double)n : P[z];
        for (int y = 0; y < nx; ++y) child[y] = m->O[y * nz + z] * bbar[y] / P[z];  /* Eq. 3 */
        uint64_t vpath = vpath_of(qpath, level, z);
        double V;
        int64_t bidx = -1;
        if (c->tr && c->tr->capture && level + 1 < cfg->depth) bidx = trace_add_belief(c->tr, child);
        if (level + 1 == cfg->depth) V = or_qmdp_value(m, c->Q, child, NULL);       /* leaf */
        else V = vnode_rec(c, child, vpath, level + 1, NULL);
        if (c->tr) {
            int64_t i = trace_add_v(c->tr);
            vrec_t *r = &c->tr->v[i];
            r->path = vpath; r->level = level + 1; r->z = z; r->f = cnt[z]; r->V = V; r->bidx = bidx;
        }
        acc += w * V;
    }
    double Qv = R + m->gamma * acc;                      /* Alg. 6 with gamma (R13) */
    if (c->tr) {
        int64_t i = trace_add_q(c->tr, n);
        qrec_t *r = &c->tr->q[i];
        r->path = qpath; r->level = level; r->action = m->action_id[a]; r->R = R; r->Q = Qv;
        for (int k = 0; k < 16; ++k) { r->P[k] = k < nz ? P[k] : 0.0; r->cnt[k] = k < nz ? cnt[k] : 0; }
        if (n > 0) {
            memcpy(&c->tr->z[i * n], zs, n);
            memcpy(&c->tr->flag[i * n], flags, n);
        }
    }
    free(bbar); free(child); free(zs); free(flags);
    return Qv;
}

/* V-node: Alg. 2 expansion over all actions, Alg. 7 V = max_a Q (ties -> lowest, R16). */
static double vnode_rec(plan_ctx *c, const double *b, uint64_t vpath, int level, double *qvals) {
    const or_model *m = c->m;
    double best = -INFINITY;
    for (int a = 0; a < m->na; ++a) {
        double q = qnode_rec(c, b, a, qpath_of(vpath, level, m->action_id[a]), level);
        if (qvals) qvals[a] = q;
        if (q > best) best = q;
    }
    return best;
}

double or_vnode_value(const or_model *m, const double *Q, const double *b, uint64_t vpath, int level,
                      const or_plan_cfg *cfg, double *qvals) {
    plan_ctx c = {m, Q, cfg, NULL};
    if (level >= cfg->depth) return or_qmdp_value(m, Q, b, NULL);
    return vnode_rec(&c, b, vpath, level, qvals);
}

int or_plan(const or_model *m, const double *Q, const double *b0, const or_plan_cfg *cfg,
            int *action, double *qroot, or_trace *trace) {
    if (!m->is_grid || cfg->depth < 0 || cfg->depth > 8 || cfg->n_samples < 0 ||
        (cfg->mode != OR_MODE_BRUTE && cfg->n_samples < 1) || cfg->n_samples > 65535)
        return OR_ERR_INVALID_ARG;
    int na = m->na;
    if (cfg->depth == 0) {                                /* plain Q_MDP on the root (R15) */
        for (int a = 0; a < na; ++a) {
            double s = 0.0;
            for (int x = 0; x < m->nx; ++x) s += b0[x] * Q[(size_t)a * m->nx + x];
            qroot[a] = s;
        }
    } else if (trace) {
        trace->nx = m->nx;
        trace->n = cfg->n_samples;
        plan_ctx c = {m, Q, cfg, trace};
        vnode_rec(&c, b0, 0, 0, qroot);
    } else {
#ifdef _OPENMP
        int th = cfg->threads > 0 ? cfg->threads : omp_get_max_threads();
#pragma omp parallel for schedule(dynamic, 1) num_threads(th)
#endif
        for (int a = 0; a < na; ++a) {
            plan_ctx c = {m, Q, cfg, NULL};
            qroot[a] = qnode_rec(&c, b0, a, qpath_of(0, 0, m->action_id[a]), 0);
        }
    }
    int arg = 0;
    for (int a = 1; a < na; ++a) if (qroot[a] > qroot[arg]) arg = a;
    *action = m->action_id[arg];
    return OR_OK;
}

int or_qnode_sample(const or_model *m, const double *b, int a, uint64_t qpath, const or_plan_cfg *cfg,
                    double *P, double *R, uint8_t *z, uint8_t *flag, uint16_t *cnt) {
    double *bbar = (double *)malloc(sizeof(double) * m->nx);
    or_predict(m, b, a, bbar);
    or_marginal(m, bbar, P);
    *R = or_belief_reward(m, b, a);
    qnode_draws(m, b, a, cfg, m->nz, P, qpath, z, flag, cnt);
    free(bbar);
    return OR_OK;
}

/* ------------------------------------------------------------------------------------------ */
/* Baselines: belief mode, MDP table lookup, A* on the mode.                   */
int or_belief_mode(const or_model *m, const double *b) {
    int arg = 0;
    for (int x = 1; x < m->nx; ++x) if (b[x] > b[arg]) arg = x;   /* ties -> lowest (R30) */
    return arg;
}

static int has_diagonal(const or_model *m) {
    for (int a = 0; a < m->na; ++a) {
        int k = m->action_id[a];
        if (k != 4 && stencil_dr(k) != 0 && stencil_dc(k) != 0) return 1;
    }
    return 0;
}

static int astar_run(const or_model *m, int start, int *first_k) {
    /* Unit-cost A* over free cells with the model's moving actions (reading R29); heuristic
     * Chebyshev when diagonals are allowed (admissible for unit diagonal cost), else Manhattan.
     * Priority (f, cell) lexicographic; neighbours expanded in ascending stencil id. */
    int nx = m->nx, W = m->W;
    int diag = has_diagonal(m);
    int gr = m->goal / W, gc = m->goal % W;
    int *g = (int *)malloc(sizeof(int) * nx), *par = (int *)malloc(sizeof(int) * nx);
    char *closed = (char *)calloc(nx, 1);
    int64_t *heap = (int64_t *)malloc(sizeof(int64_t) * (size_t)nx * 9 + 16);
    int hn = 0;
    for (int x = 0; x < nx; ++x) { g[x] = -1; par[x] = -1; }
#define HKEY(f, x) (((int64_t)(f) << 32) | (int64_t)(x))
#define HEUR(x) (diag ? (abs((x) / W - gr) > abs((x) % W - gc) ? abs((x) / W - gr) : abs((x) % W - gc)) \
                      : abs((x) / W - gr) + abs((x) % W - gc))
    g[start] = 0;
    heap[hn++] = HKEY(HEUR(start), start);
    int found = 0;
    while (hn > 0) {
        int64_t top = heap[0];
        heap[0] = heap[--hn];
        for (int i = 0;;) {                                /* sift down */
            int l = 2 * i + 1, r = l + 1, s = i;
            if (l < hn && heap[l] < heap[s]) s = l;
            if (r < hn && heap[r] < heap[s]) s = r;
            if (s == i) break;
            int64_t tmp = heap[i]; heap[i] = heap[s]; heap[s] = tmp; i = s;
        }
        int x = (int)(top & 0xFFFFFFFF);
        if (closed[x]) continue;
        closed[x] = 1;
        if (x == m->goal) { found = 1; break; }
        for (int a = 0; a < m->na; ++a) {
            int k = m->action_id[a];
            if (k == 4) continue;
            int o, y = grid_neighbour(m, x, k, &o);
            if (o || closed[y]) continue;
            if (g[y] < 0 || g[x] + 1 < g[y]) {
                g[y] = g[x] + 1; par[y] = x;
                int i = hn++;
                heap[i] = HKEY(g[y] + HEUR(y), y);
                while (i > 0 && heap[(i - 1) / 2] > heap[i]) {   /* sift up */
                    int p = (i - 1) / 2;
                    int64_t tmp = heap[i]; heap[i] = heap[p]; heap[p] = tmp; i = p;
                }
            }
        }
    }
#undef HKEY
#undef HEUR
    int len = -1;
    if (found) {
        len = g[m->goal];
        int y = m->goal;
        if (y != start) {
            while (par[y] != start) y = par[y];
            int dr = y / W - start / W, dc = y % W - start % W;
            *first_k = 3 * (dr + 1) + (dc + 1);
        } else *first_k = 4;
    }
    free(g); free(par); free(closed); free(heap);
    return len;
}

int or_astar_length(const or_model *m, int start) {
    int k;
    return astar_run(m, start, &k);
}

int or_astar_action(const or_model *m, int start) {
    int k = 4;
    if (astar_run(m, start, &k) < 0) k = 4;
    for (int a = 0; a < m->na; ++a) if (m->action_id[a] == k) return k;
    return m->action_id[0];
}

/* Alg. 4 literal: x ~ b, x' ~ P(x'|x,a) (clamped T), z ~ P(z|x'),
 * using Philox words 1..3 of one call. */
int or_ancestral_sample(const or_model *m, const double *b, int a, const uint32_t ctr[4],
                        const uint32_t key[2]) {
    uint32_t w[4];
    or_philox4x32_10(ctr, key, w);
    int x = or_inverse_cdf(b, m->nx, or_uniform(w[1]), NULL);
    int e0 = m->t_start[x * m->na + a], e1 = m->t_start[x * m->na + a + 1];
    double *p = (double *)malloc(sizeof(double) * (e1 - e0));
    for (int e = e0; e < e1; ++e) p[e - e0] = m->t_p[e];
    int xp = m->t_y[e0 + or_inverse_cdf(p, e1 - e0, or_uniform(w[2]), NULL)];
    free(p);
    return or_inverse_cdf(&m->O[xp * m->nz], m->nz, or_uniform(w[3]), NULL);
}

/* ------------------------------------------------------------------------------------------ */
/* Closed-loop episodes (Alg. 1 outer loop PAPER.md:149-165; Eq. 1 return PAPER.md:36-42;
 * termination/collision readings R26/R27; environment draws per Appendix A.2). */
int or_run_episode(const or_model *m, const double *Q, const double *b0, const or_episode_cfg *cfg,
                   or_episode_record *rec, int32_t *log_a, int32_t *log_z, int32_t *log_x) {
    if (!m->is_grid) return OR_ERR_INVALID_ARG;
    int nx = m->nx, na = m->na;
    double *b = (double *)malloc(sizeof(double) * nx), *bn = (double *)malloc(sizeof(double) * nx);
    double *qroot = (double *)malloc(sizeof(double) * na);
    memcpy(b, b0, sizeof(double) * nx);
    uint32_t key[2] = {cfg->seed, cfg->episode}, w[4];
    uint32_t ctr0[4] = {0, 0, 0, 0};
    or_philox4x32_10(ctr0, key, w);
    int x = or_inverse_cdf(b0, nx, or_uniform(w[2]), NULL);      /* x0 ~ b0 */
    memset(rec, 0, sizeof(*rec));
    rec->x0 = x;
    rec->outcome = 2;
    double disc = 1.0;
    int streak = 0, s;
    for (s = 0; s < cfg->max_steps; ++s) {
        int a_id;
        if (cfg->planner == OR_PLANNER_QVTS) {
            or_plan_cfg pc;
            memset(&pc, 0, sizeof(pc));
            pc.depth = cfg->depth; pc.n_samples = cfg->n_samples; pc.mode = OR_MODE_FREQ;
            pc.seed = cfg->seed; pc.step = (uint32_t)s; pc.episode = cfg->episode; pc.threads = 1;
            or_plan(m, Q, b, &pc, &a_id, qroot, NULL);
        } else if (cfg->planner == OR_PLANNER_MDP) {
            int xm = or_belief_mode(m, b), arg = 0;
            for (int a = 1; a < na; ++a)
                if (Q[(size_t)a * nx + xm] > Q[(size_t)arg * nx + xm]) arg = a;
            a_id = m->action_id[arg];
        } else {
            a_id = or_astar_action(m, or_belief_mode(m, b));
        }
        int a = 0;
        while (m->action_id[a] != a_id) ++a;
        uint32_t ctr[4] = {0, 0, 0, (uint32_t)s};
        or_philox4x32_10(ctr, key, w);
        /* true motion y ~ T'(x,a,.) in stencil order; blocked -> collision, stay */
        int k = or_inverse_cdf(&m->Tp[((size_t)x * na + a) * 9], 9, or_uniform(w[0]), NULL);
        int xn = x;
        if (k != 4) {
            int o, y = grid_neighbour(m, x, k, &o);
            if (o) rec->collisions++;
            else xn = y;
        }
        int z = or_inverse_cdf(&m->O[xn * m->nz], m->nz, or_uniform(w[1]), NULL);
        rec->disc_return += disc * m->R[x * na + a];
        disc *= m->gamma;
        double pz;
        int st = or_belief_update(m, b, a, z, bn, &pz);
        if (log_a) log_a[s] = a_id;
        if (log_z) log_z[s] = z;
        if (log_x) log_x[s] = xn;
        x = xn;
        if (st != OR_OK) { rec->outcome = 3; ++s; break; }
        memcpy(b, bn, sizeof(double) * nx);
        streak = (a_id == 4) ? streak + 1 : 0;
        if (cfg->stop_patience > 0 && streak >= cfg->stop_patience) {
            rec->outcome = (x == m->goal) ? 0 : 1;
            ++s;
            break;
        }
    }
    rec->steps = s;
    rec->x_final = x;
    free(b); free(bn); free(qroot);
    return OR_OK;
}

/* ------------------------------------------------------------------------------------------ */
/* Anytime best-first QVTS (Alg. 1-7, Eq. 8).          */
/* Nodes live in flat arrays; V-node i carries its belief, (U, L, H, E) and its Q-children     */
/* [q0, q0 + na); Q-node j carries (R, U, L, H, E) and its V-children [c0, c0 + nc).           */
void or_bf_q_update(double R, double gamma, int nc, const double *w, const double *U, const double *L,
                    const double *H, const int *E, double *UQ, double *LQ, double *HQ, int *EQ) {
    double su = 0.0, sl = 0.0, bh = 0.0;
    int bc = 0;
    for (int c = 0; c < nc; ++c) {
        su += w[c] * U[c];
        sl += w[c] * L[c];
        double h = gamma * w[c] * H[c];                 /* Alg. 6: gamma x weight x heuristic */
        if (c == 0 || h > bh) { bh = h; bc = c; }
    }
    *UQ = R + gamma * su;                               /* Alg. 6 with gamma (R13, Eq. 2)     */
    *LQ = R + gamma * sl;
    *HQ = bh;
    *EQ = E[bc];
}

void or_bf_v_update(int na, const double *UQ, const double *LQ, const double *HQ, const int *EQ,
                    double *U, double *L, double *H, int *E) {
    int bq = 0;
    double bl = LQ[0];
    for (int a = 1; a < na; ++a) {
        if (UQ[a] > UQ[bq]) bq = a;                     /* H(b,a) = 1 at argmax U_Q (Sec. IV-C) */
        if (LQ[a] > bl) bl = LQ[a];
    }
    *U = UQ[bq];
    *L = bl;
    *H = HQ[bq];
    *E = EQ[bq];
}

typedef struct {
    double *b;
    uint64_t path;
    int depth, pq, z, f, q0, E;
    double w, U, L, H;
} bf_v;
typedef struct {
    int pv, a, c0, nc, E;
    double R, U, L, H;
} bf_q;
struct or_bf_tree {
    const or_model *m;
    int na, root;
    bf_v *v;
    bf_q *q;
    int nv, nq, cap_v, cap_q;
    int action, stop, n_exp, subs, mism;
    uint64_t *exp_path;
    double *rootU, *rootL;
};

static double bf_dot_max(const double *A, int n, int nx, const double *b, int *arg) {
    double best = 0.0;
    int ba = 0;
    for (int k = 0; k < n; ++k) {
        double s = 0.0;
        for (int x = 0; x < nx; ++x) s += A[(size_t)k * nx + x] * b[x];
        if (k == 0 || s > best) { best = s; ba = k; }
    }
    if (arg) *arg = ba;
    return best;
}

static int bf_new_v(or_bf_tree *t) {
    if (t->nv == t->cap_v) {
        t->cap_v *= 2;
        t->v = (bf_v *)realloc(t->v, sizeof(bf_v) * t->cap_v);
    }
    memset(&t->v[t->nv], 0, sizeof(bf_v));
    return t->nv++;
}

static void bf_update_q(or_bf_tree *t, int j) {
    bf_q *q = &t->q[j];
    int nc = q->nc;
    double w[16], U[16], L[16], H[16];
    int E[16];
    for (int c = 0; c < nc; ++c) {
        const bf_v *v = &t->v[q->c0 + c];
        w[c] = v->w; U[c] = v->U; L[c] = v->L; H[c] = v->H; E[c] = v->E;
    }
    or_bf_q_update(q->R, t->m->gamma, nc, w, U, L, H, E, &q->U, &q->L, &q->H, &q->E);
}

static void bf_update_v(or_bf_tree *t, int i) {
    bf_v *v = &t->v[i];
    double UQ[9], LQ[9], HQ[9];
    int EQ[9];
    for (int a = 0; a < t->na; ++a) {
        const bf_q *q = &t->q[v->q0 + a];
        UQ[a] = q->U; LQ[a] = q->L; HQ[a] = q->H; EQ[a] = q->E;
    }
    or_bf_v_update(t->na, UQ, LQ, HQ, EQ, &v->U, &v->L, &v->H, &v->E);
}

/* Alg. 5: a new leaf V-node with U = V_FIB(b), L = V_PBVI(b), H = U - L, E = self. */
static void bf_leaf(or_bf_tree *t, int i, const double *aU, int nU, const double *aL, int nL, int max_depth) {
    bf_v *v = &t->v[i];
    int nx = t->m->nx;
    v->U = bf_dot_max(aU, nU, nx, v->b, NULL);
    v->L = bf_dot_max(aL, nL, nx, v->b, NULL);
    v->H = v->depth >= max_depth ? 0.0 : v->U - v->L;    /* terminal leaves (reading B5) */
    v->E = i;
    v->q0 = -1;
}

/* Alg. 2 + Alg. 3: all |A| Q-nodes of leaf i, one child per unique sampled z (or every z with
 * P > 0 in EXACT mode), then the Alg. 6 / Alg. 7 updates of i. */
static void bf_expand(or_bf_tree *t, int i, const double *aU, int nU, const double *aL, int nL,
                      const or_plan_cfg *pcfg, int max_depth) {
    const or_model *m = t->m;
    int nx = m->nx, nz = m->nz, na = t->na, n = pcfg->n_samples;
    double *bbar = (double *)malloc(sizeof(double) * nx);
    uint8_t *zs = (uint8_t *)calloc(n > 0 ? n : 1, 1), *fl = (uint8_t *)calloc(n > 0 ? n : 1, 1);
    if (t->nq + na > t->cap_q) {
        while (t->nq + na > t->cap_q) t->cap_q *= 2;
        t->q = (bf_q *)realloc(t->q, sizeof(bf_q) * t->cap_q);
    }
    int q0 = t->nq;
    t->nq += na;
    t->v[i].q0 = q0;
    for (int a = 0; a < na; ++a) {
        const double *b = t->v[i].b;
        uint64_t vpath = t->v[i].path;
        int depth = t->v[i].depth;
        uint64_t qpath = qpath_of(vpath, depth, m->action_id[a]);
        double P[16];
        uint16_t cnt[16];
        or_predict(m, b, a, bbar);
        or_marginal(m, bbar, P);
        bf_q *q = &t->q[q0 + a];
        q->pv = i; q->a = a;
        q->R = or_belief_reward(m, b, a);
        if (pcfg->mode == OR_MODE_EXACT) { for (int z = 0; z < nz; ++z) cnt[z] = 0; }
        else qnode_draws(m, b, a, pcfg, nz, P, qpath, zs, fl, cnt);
        q->c0 = t->nv;
        q->nc = 0;
        for (int z = 0; z < nz; ++z) {
            int take = pcfg->mode == OR_MODE_EXACT ? (P[z] > OR_ZERO_LIK) : (cnt[z] > 0);
            if (!take) continue;
            int c = bf_new_v(t);
            bf_v *v = &t->v[c];
            v->b = (double *)malloc(sizeof(double) * nx);
            for (int y = 0; y < nx; ++y) v->b[y] = m->O[y * nz + z] * bbar[y] / P[z];   /* Eq. 3 */
            v->path = vpath_of(qpath, depth, z);
            v->depth = depth + 1;
            v->pq = q0 + a;
            v->z = z;
            v->f = cnt[z];
            v->w = pcfg->mode == OR_MODE_EXACT ? P[z] : (double)cnt[z] / (double)n;
            bf_leaf(t, c, aU, nU, aL, nL, max_depth);
            t->q[q0 + a].nc++;
        }
        bf_update_q(t, q0 + a);
    }
    bf_update_v(t, i);
    free(bbar); free(zs); free(fl);
}

/* Admissible descent: at every decision the chosen child is within `tol` of the rule's best. */
static int bf_admissible(const or_bf_tree *t, uint64_t path, double tol) {
    int i = t->root;
    for (;;) {
        const bf_v *v = &t->v[i];
        if (v->q0 < 0) return v->path == path ? i : -1;
        int lvl = v->depth;
        int aid = (int)((path >> (8 * lvl)) & 15) - 1;
        int z = (int)((path >> (8 * lvl + 4)) & 15);
        int a = -1;
        for (int k = 0; k < t->na; ++k) if (t->m->action_id[k] == aid) a = k;
        if (a < 0) return -1;
        double bu = -INFINITY;
        for (int k = 0; k < t->na; ++k) bu = fmax(bu, t->q[v->q0 + k].U);
        const bf_q *q = &t->q[v->q0 + a];
        if (q->U < bu - tol) return -1;
        double bh = -INFINITY;
        int c = -1;
        for (int k = 0; k < q->nc; ++k) {
            const bf_v *ch = &t->v[q->c0 + k];
            bh = fmax(bh, t->m->gamma * ch->w * ch->H);
            if (ch->z == z) c = q->c0 + k;
        }
        if (c < 0 || t->m->gamma * t->v[c].w * t->v[c].H < bh - tol) return -1;
        i = c;
    }
}

/* Alg. 1 inner loop from the current root: expansions until planningFinished(), then
 * getOptimalAction.  Counters and traces are per call. */
static void bf_run(or_bf_tree *t, const double *alphaU, int nU, const double *alphaL, int nL, const int *actL,
                   const or_plan_cfg *pcfg, const or_bf_cfg *bcfg) {
    const or_model *m = t->m;
    free(t->exp_path); free(t->rootU); free(t->rootL);
    t->exp_path = (uint64_t *)calloc(bcfg->expansions + 1, sizeof(uint64_t));
    t->rootU = (double *)calloc(bcfg->expansions + 1, sizeof(double));
    t->rootL = (double *)calloc(bcfg->expansions + 1, sizeof(double));
    t->n_exp = 0; t->subs = 0; t->mism = 0; t->stop = 0;
    const int r = t->root;
    for (;;) {
        t->rootU[t->n_exp] = t->v[r].U;
        t->rootL[t->n_exp] = t->v[r].L;
        if (t->n_exp >= bcfg->expansions) { t->stop = 0; break; }          /* planningFinished() */
        if (t->v[r].U - t->v[r].L <= bcfg->gap_tol) { t->stop = 1; break; }
        int e = t->v[r].E;                                 /* findVNodeToExpand() = root.E */
        if (bcfg->n_replay > t->n_exp) {
            int g = bf_admissible(t, bcfg->replay_path[t->n_exp], bcfg->replay_tol);
            if (g < 0) t->mism++;
            else if (g != e) { t->subs++; e = g; }
        }
        if (t->v[e].depth >= bcfg->max_depth) { t->stop = 2; break; }
        t->exp_path[t->n_exp++] = t->v[e].path;
        bf_expand(t, e, alphaU, nU, alphaL, nL, pcfg, bcfg->max_depth);     /* v.expand() */
        for (int p = t->v[e].pq; p >= 0; p = t->v[t->q[p].pv].pq) {         /* p.update() to the root */
            bf_update_q(t, p);
            bf_update_v(t, t->q[p].pv);
        }
    }
    /* getOptimalAction: max L_Q, ties by U_Q then index (SPEC plan); an unexpanded root takes the
     * action of its PBVI arg-max vector. */
    if (t->v[r].q0 < 0) {
        int arg;
        bf_dot_max(alphaL, nL, m->nx, t->v[r].b, &arg);
        t->action = actL ? actL[arg] : 0;
    } else {
        int best = 0;
        for (int a = 1; a < t->na; ++a) {
            const bf_q *q = &t->q[t->v[r].q0 + a], *bq = &t->q[t->v[r].q0 + best];
            if (q->L > bq->L || (q->L == bq->L && q->U > bq->U)) best = a;
        }
        t->action = m->action_id[best];
    }
}

or_bf_tree *or_bf_plan(const or_model *m, const double *alphaU, int nU, const double *alphaL, int nL,
                       const int *actL, const double *b0, const or_plan_cfg *pcfg, const or_bf_cfg *bcfg) {
    if (bcfg->max_depth < 1 || bcfg->max_depth > 8 || nU < 1 || nL < 1 || bcfg->expansions < 0) return NULL;
    or_bf_tree *t = (or_bf_tree *)calloc(1, sizeof(or_bf_tree));
    t->m = m;
    t->na = m->na;
    t->cap_v = 64; t->cap_q = 64;
    t->v = (bf_v *)malloc(sizeof(bf_v) * t->cap_v);
    t->q = (bf_q *)malloc(sizeof(bf_q) * t->cap_q);
    int r = bf_new_v(t);                                   /* Alg. 1: s = QVSearchTree(b0) */
    t->root = r;
    t->v[r].b = (double *)malloc(sizeof(double) * m->nx);
    memcpy(t->v[r].b, b0, sizeof(double) * m->nx);
    t->v[r].pq = -1;
    t->v[r].f = pcfg->n_samples;
    t->v[r].w = 1.0;
    bf_leaf(t, r, alphaU, nU, alphaL, nL, bcfg->max_depth);
    bf_run(t, alphaU, nU, alphaL, nL, actL, pcfg, bcfg);
    return t;
}

int or_bf_continue(or_bf_tree *t, const double *alphaU, int nU, const double *alphaL, int nL, const int *actL,
                   const or_plan_cfg *pcfg, const or_bf_cfg *bcfg) {
    if (bcfg->max_depth < 1 || bcfg->max_depth > 8 || bcfg->expansions < 0) return OR_ERR_INVALID_ARG;
    bf_run(t, alphaU, nU, alphaL, nL, actL, pcfg, bcfg);
    return OR_OK;
}

/* s.update(a, z) (Alg. 1; SPEC advance_root): when the root's Q-node for stencil id a_id has a
 * child with observation z, that V-node becomes the root and keeps its subtree; its paths lose
 * their first byte and depths drop by one (so later draws are keyed relative to the new root),
 * every node outside it is discarded (depth -1).  Returns 1 on reuse, 0 when z was not sampled
 * (the caller builds a fresh root from Eq. 3). */
int or_bf_advance(or_bf_tree *t, int a_id, int z) {
    const bf_v *root = &t->v[t->root];
    if (root->q0 < 0) return 0;
    int a = -1;
    for (int k = 0; k < t->na; ++k) if (t->m->action_id[k] == a_id) a = k;
    if (a < 0) return 0;
    const bf_q *q = &t->q[root->q0 + a];
    int c = -1;
    for (int i = 0; i < q->nc; ++i) if (t->v[q->c0 + i].z == z) c = q->c0 + i;
    if (c < 0) return 0;
    /* subtree membership: walk each node's parent chain up to depth 1 */
    for (int i = 0; i < t->nv; ++i) {
        bf_v *v = &t->v[i];
        if (v->depth < 1) { v->depth = -1; continue; }
        int j = i;
        while (t->v[j].depth > 1) j = t->q[t->v[j].pq].pv;
        if (j != c) { v->depth = -1; continue; }
    }
    for (int i = 0; i < t->nv; ++i) {
        bf_v *v = &t->v[i];
        if (v->depth < 0) continue;
        v->depth -= 1;
        v->path >>= 8;
    }
    t->v[c].pq = -1;
    t->v[c].w = 1.0;
    t->root = c;
    return 1;
}

void or_bf_free(or_bf_tree *t) {
    if (!t) return;
    for (int i = 0; i < t->nv; ++i) free(t->v[i].b);
    free(t->v); free(t->q); free(t->exp_path); free(t->rootU); free(t->rootL); free(t);
}
void or_bf_summary(const or_bf_tree *t, int *action, int *stop, int *n_exp, int *n_v, int *subs, int *mism) {
    *action = t->action; *stop = t->stop; *n_exp = t->n_exp; *n_v = t->nv; *subs = t->subs; *mism = t->mism;
}
void or_bf_root(const or_bf_tree *t, double *U, double *L, double *UQ, double *LQ) {
    const bf_v *r = &t->v[t->root];
    *U = r->U;
    *L = r->L;
    for (int a = 0; a < t->na; ++a) {
        int ok = r->q0 >= 0;
        if (UQ) UQ[a] = ok ? t->q[r->q0 + a].U : NAN;
        if (LQ) LQ[a] = ok ? t->q[r->q0 + a].L : NAN;
    }
}
int or_bf_root_index(const or_bf_tree *t) { return t->root; }
void or_bf_belief(const or_bf_tree *t, int i, double *out) { memcpy(out, t->v[i].b, sizeof(double) * t->m->nx); }
void or_bf_vnode(const or_bf_tree *t, int i, uint64_t *path, int *depth, int *f, double *w, double *U,
                 double *L, double *H, int *E, int *expanded) {
    const bf_v *v = &t->v[i];
    *path = v->path; *depth = v->depth; *f = v->f; *w = v->w; *U = v->U; *L = v->L; *H = v->H; *E = v->E;
    *expanded = v->q0 >= 0;
}
uint64_t or_bf_expanded(const or_bf_tree *t, int k) { return t->exp_path[k]; }
void or_bf_root_trace(const or_bf_tree *t, int k, double *U, double *L) { *U = t->rootU[k]; *L = t->rootL[k]; }
