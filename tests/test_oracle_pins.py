"""Pins of the fp64 CPU oracle against values and properties the paper and mathematics fix
(SURVEY.md §8(c) c.4).  CPU only."""
import json
import os
from collections import deque

import numpy as np
import pytest

import oracle as O
import workloads as W

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "pins.json")))


def open3x3(goal=0, blocked=()):
    occ = np.zeros(9, np.uint8)
    for b in blocked:
        occ[b] = 1
    return W.GridMap(3, 3, occ, goal)


def dense_T(m):
    T = np.zeros((m.nx, m.na, m.nx))
    for x in range(m.nx):
        for a in range(m.na):
            for y in range(m.nx):
                T[x, a, y] = m.T(x, a, y)
    return T


# ---- P1 RNG ------------------------------------------------------------------------------
def test_philox_known_answers():
    for v in GOLD["philox_kat"]["vectors"]:
        ctr = [int(h, 16) for h in v["ctr"]]
        key = [int(h, 16) for h in v["key"]]
        out = O.philox(ctr, key)
        assert [f"{w:08x}" for w in out] == v["out"]


def test_uniform_and_inverse_cdf():
    assert O.uniform(0) == 0.5 * 2.0 ** -24
    assert O.uniform(0xFFFFFFFF) == 1.0 - 0.5 * 2.0 ** -24
    # strict '<' never picks a zero-weight category (Appendix A.5)
    p = [0.0, 0.5, 0.0, 0.5]
    assert O.inverse_cdf(p, 1e-9)[0] == 1
    assert O.inverse_cdf(p, 0.5)[0] == 3
    assert O.inverse_cdf(p, 0.4999999)[0] == 1
    assert O.inverse_cdf(p, 0.4999999)[1]       # within 1e-6 of the boundary -> flagged
    assert not O.inverse_cdf(p, 0.3)[1]


# ---- P2 model tables ---------------------------------------------------------------------
def test_transition_examples():
    g = GOLD["transition_up_open"]
    m = O.Model.grid(open3x3(goal=8))
    up = m.action_ids.index(1)
    assert m.T(4, up, 1) == pytest.approx(g["T_up_N1"], abs=1e-15)
    assert m.T(4, up, 4) == pytest.approx(g["T_up_stay"], abs=1e-15)
    assert m.T(4, up, 0) == pytest.approx(g["T_up_N0"], abs=1e-15)
    assert m.T(4, up, 2) == pytest.approx(g["T_up_N2"], abs=1e-15)
    mb = O.Model.grid(open3x3(goal=8, blocked=(1,)))
    assert mb.T(4, up, 4) == pytest.approx(g["T_up_stay_N1_blocked"], abs=1e-15)
    assert mb.T(4, up, 0) == pytest.approx(0.05, abs=1e-15)
    # diagonal laterals are ring neighbours (R3): up-left (0) -> {3, 1}
    ul = m.action_ids.index(0)
    assert m.T(4, ul, 3) == pytest.approx(0.05) and m.T(4, ul, 1) == pytest.approx(0.05)
    assert m.T(4, ul, 0) == pytest.approx(0.8) and m.T(4, ul, 4) == pytest.approx(0.1)
    # stay is deterministic (R2)
    assert m.T(4, m.action_ids.index(4), 4) == 1.0


def test_table_invariants_random_map():
    gm = W.random_map(9, 11, 0.25, seed=7)
    m = O.Model.grid(gm)
    T = dense_T(m)
    assert np.allclose(T.sum(axis=2), 1.0, atol=1e-12)
    occ = gm.occupancy.astype(bool)
    free = ~occ
    # T(x, a, y) = 0 for occupied y and free x
    assert np.all(T[np.ix_(free, np.arange(m.na), occ)] == 0.0)
    Ot = m.O_table()
    assert np.allclose(Ot.sum(axis=1), 1.0, atol=1e-12)


def test_observation_examples():
    g = GOLD["observation"]
    m = O.Model.grid(open3x3(goal=8))
    assert m.sig(4) == 0
    assert m.O(4, 0) == pytest.approx(g["all_free_z0"], abs=1e-15)
    assert m.O(4, 1) == pytest.approx(g["all_free_z1"], abs=1e-15)
    # corner (0,0): up (bit0) and left (bit1) off-map read occupied
    assert m.sig(0) == 0b0011
    assert m.sig(8) == 0b1100
    # acc = 1 -> exactly one observation with likelihood 1
    m1 = O.Model.grid(open3x3(goal=8), acc=1.0)
    row = np.array([m1.O(4, z) for z in range(16)])
    assert row[0] == 1.0 and row.sum() == 1.0


def test_reward_examples():
    m = O.Model.grid(open3x3(goal=0))
    R = [m.R(4, a) for a in range(9)]
    assert np.allclose(R, GOLD["reward_centre_goal_topleft_3x3"]["R"], atol=1e-15)
    assert m.R(0, 4) == 0.0            # stay at goal
    assert m.R(8, 4) == -2.0           # stay off goal


def test_reward_collision_cases():
    """PAPER.md:338-355 by hand: R(x,a) = sum_y r(y) T'(x,a,y) with the pre-clamp T', r = -2 on an
    occupied or off-map target, -1 on a free non-goal cell; laterals are the ring neighbours (R3)."""
    m = O.Model.grid(open3x3(goal=8))
    # corner 0, action 0 (up-left): intended and both laterals (1 up, 3 left) leave the map
    assert m.R(0, 0) == pytest.approx(0.8 * -2 + 0.1 * -1 + 0.05 * -2 + 0.05 * -2, abs=1e-15)
    m = O.Model.grid(open3x3(goal=8, blocked=(4,)))
    # cell 1, action 7 (down) into the occupied centre; laterals 8 -> cell 5, 6 -> cell 3 are free
    assert m.R(1, 7) == pytest.approx(0.8 * -2 + 0.1 * -1 + 0.05 * -1 + 0.05 * -1, abs=1e-15)
    # cell 7, action 5 (right) onto the goal 8: laterals 2 -> cell 5 (free), 8 -> off the map
    assert m.R(7, 5) == pytest.approx(0.8 * 0 + 0.1 * -1 + 0.05 * -1 + 0.05 * -2, abs=1e-15)


# ---- P3 / P4 / P11 Eq. 3 -------------------------------------------------------------------
def test_bayes_two_state_example():
    T = np.zeros((2, 1, 2)); T[0, 0, 0] = 1; T[1, 0, 1] = 1
    Om = np.array([[0.9, 0.1], [0.2, 0.8]])
    R = np.zeros((2, 1))
    m = O.Model.dense(T, Om, R, 0.95)
    post, p = m.belief_update(np.array([0.5, 0.5]), 0, 0)
    g = GOLD["bayes_two_state"]
    assert p == pytest.approx(g["p_obs"], abs=1e-15)
    assert np.allclose(post, g["posterior"], atol=1e-15)
    assert m.marginal(m.predict(np.array([0.5, 0.5]), 0)) == pytest.approx([0.55, 0.45])


def test_bayes_point_mass_chain_and_uniform_invariance():
    T = np.zeros((2, 1, 2)); T[0, 0, 1] = 1; T[1, 0, 1] = 1
    Om = np.array([[0.7, 0.3], [0.5, 0.5]])
    m = O.Model.dense(T, Om, np.zeros((2, 1)), 0.9)
    post, _ = m.belief_update(np.array([1.0, 0.0]), 0, 0)
    assert np.array_equal(post, [0.0, 1.0])
    T2 = np.zeros((3, 1, 3))
    for i in range(3):
        T2[i, 0, i] = 1
    m2 = O.Model.dense(T2, np.full((3, 2), 0.5), np.zeros((3, 1)), 0.9)
    b = np.ones(3) / 3
    post, _ = m2.belief_update(b, 0, 1)
    assert np.allclose(post, b, atol=1e-15)


def test_zero_likelihood():
    T = np.zeros((2, 1, 2)); T[0, 0, 0] = 1; T[1, 0, 1] = 1
    Om = np.array([[1.0, 0.0], [1.0, 0.0]])
    m = O.Model.dense(T, Om, np.zeros((2, 1)), 0.9)
    with pytest.raises(O.OracleError) as e:
        m.belief_update(np.array([0.5, 0.5]), 0, 1)
    assert e.value.code == O.ERR_ZERO_LIKELIHOOD


def test_belief_reward_example():
    T = np.zeros((3, 1, 3))
    for i in range(3):
        T[i, 0, i] = 1
    m = O.Model.dense(T, np.ones((3, 1)), np.array([[-2.0], [-1.0], [0.0]]), 0.9)
    assert m.belief_reward(np.array([0.2, 0.3, 0.5]), 0) == pytest.approx(GOLD["belief_reward"]["value"], abs=1e-15)


@pytest.mark.parametrize("seed", [1, 2])
def test_predict_matches_dense_product_and_total_probability(seed):
    gm = W.random_map(7, 9, 0.2, seed=seed)
    m = O.Model.grid(gm)
    T = dense_T(m)
    b = W.random_belief(gm, seed + 10)
    for a in range(m.na):
        bbar = m.predict(b, a)
        assert np.allclose(bbar, T[:, a, :].T @ b, atol=1e-15)
        assert bbar.sum() == pytest.approx(1.0, abs=1e-12)
        P = m.marginal(bbar)
        assert P.sum() == pytest.approx(1.0, abs=1e-12)
        recon = np.zeros(m.nx)
        for z in range(16):
            post, p = m.belief_update(b, a, z)
            assert p == pytest.approx(P[z], abs=1e-15)
            assert post.sum() == pytest.approx(1.0, abs=1e-12)           # P11
            assert np.all(post[gm.occupancy == 1] == 0.0)                # P11 support
            recon += p * post
        assert np.allclose(recon, bbar, atol=1e-12)                      # P4


# ---- P5 value iteration --------------------------------------------------------------------
@pytest.mark.parametrize("L", [3, 6])
def test_vi_corridor_closed_form(L):
    m = O.Model.grid(W.corridor(L), action_mask=W.A9, p_int=1.0, p_stay=0.0, p_lat=0.0)
    st, V, Q, sweeps, res = m.value_iteration(1e-9)
    assert st == O.OK and res < 1e-9
    assert np.allclose(V, GOLD["corridor_vi"][f"L{L}"], atol=1e-8)


def test_vi_constant_reward_dense():
    rng = np.random.default_rng(0)
    T = rng.random((4, 2, 4)); T /= T.sum(axis=2, keepdims=True)
    m = O.Model.dense(T, np.ones((4, 1)), np.full((4, 2), -3.0), 0.9)
    st, V, Q, _, res = m.value_iteration(1e-11)
    assert st == O.OK
    assert np.allclose(V, -3.0 / (1 - 0.9), atol=1e-9)


def test_vi_fixed_point_random_map():
    gm = W.random_map(20, 23, 0.2, seed=5)
    m = O.Model.grid(gm, action_mask=W.A8)
    st, V, Q, sweeps, res = m.value_iteration(1e-9)
    assert st == O.OK and res < 1e-9 and sweeps > 50
    free = gm.occupancy == 0
    assert np.allclose(Q.max(axis=0)[free], V[free], atol=2e-8)
    T = dense_T(m)
    R = m.R_table()
    for a in range(m.na):   # Q = R + gamma T V on free cells
        assert np.allclose((R[a] + 0.95 * T[:, a, :] @ V)[free], Q[a][free], atol=1e-12)
    assert np.all(V[free] < 0) and V[gm.goal] > -12


# ---- P6 / P7 / P8 plan step -----------------------------------------------------------------
def _small(seed=3, acc=0.95, mask=W.A4, H=5, Wd=6):
    gm = W.random_map(H, Wd, 0.15, seed=seed)
    m = O.Model.grid(gm, action_mask=mask, acc=acc)
    st, V, Q, _, _ = m.value_iteration(1e-10)
    return gm, m, Q


def test_depth0_is_qmdp():
    gm, m, Q = _small()
    b = W.random_belief(gm, 1)
    r = m.plan(Q, b, depth=0, n=4)
    assert np.allclose(r.qroot, Q @ b, atol=1e-14)
    assert r.action == m.action_ids[int(np.argmax(Q @ b))]


def _dense_brute(T, Om, R, Q, gamma, b, depth):
    """Eq. 2 written with dense matrices (brute force over all z, tiny inputs)."""
    na = T.shape[1]
    qs = []
    for a in range(na):
        bbar = T[:, a, :].T @ b
        val = R[a] @ b
        for z in range(Om.shape[1]):
            pz = Om[:, z] @ bbar
            if pz <= 1e-300:
                continue
            child = Om[:, z] * bbar / pz
            if depth == 1:
                v = (Q @ child).max()
            else:
                v = max(_dense_brute(T, Om, R, Q, gamma, child, depth - 1))
            val += gamma * pz * v
        qs.append(val)
    return qs


def test_depth1_closed_form_unnormalised():
    gm, m, Q = _small(seed=4, mask=W.A8)
    T, Om, R = dense_T(m), m.O_table(), m.R_table()
    b = W.uniform_belief(gm)
    r = m.plan(Q, b, depth=1, n=4, mode=O.MODE_BRUTE)
    for a in range(m.na):
        bbar = T[:, a, :].T @ b
        expect = R[a] @ b + 0.95 * sum((Q @ (Om[:, z] * bbar)).max() for z in range(16))
        assert r.qroot[a] == pytest.approx(expect, abs=1e-12)


@pytest.mark.parametrize("depth", [1, 2])
def test_brute_force_matches_dense_recursion(depth):
    gm, m, Q = _small(seed=6, acc=0.8, H=4, Wd=4)
    T, Om, R = dense_T(m), m.O_table(), m.R_table()
    b = W.random_belief(gm, 3)
    r = m.plan(Q, b, depth=depth, n=4, mode=O.MODE_BRUTE)
    assert np.allclose(r.qroot, _dense_brute(T, Om, R, Q, 0.95, b, depth), atol=1e-12)


def test_exact_mode_with_covering_samples_equals_brute():
    gm, m, Q = _small(seed=6, acc=0.75, H=4, Wd=4)
    b = W.uniform_belief(gm)
    brute = m.plan(Q, b, depth=2, n=4, mode=O.MODE_BRUTE)
    ex = m.plan(Q, b, depth=2, n=4096, mode=O.MODE_EXACT, trace=True)
    covered = (ex.trace.q_cnt > 0) | (ex.trace.q_P <= 1e-300)
    assert covered.all()
    assert np.allclose(ex.qroot, brute.qroot, atol=1e-12)
    fr = m.plan(Q, b, depth=2, n=4096, mode=O.MODE_FREQ)
    assert np.allclose(fr.qroot, brute.qroot, atol=0.05)   # O(n^-1/2) sampling gap (R31)


# ---- P9 sampling distribution ---------------------------------------------------------------
def test_sampling_frequencies_and_ancestral_equivalence():
    gm = W.random_map(8, 8, 0.2, seed=2)
    m = O.Model.grid(gm, action_mask=W.A9, acc=0.8)
    b = W.random_belief(gm, 4)
    a = 1
    n = 60000
    P, R, z, flag, cnt = m.qnode_sample(b, a, qpath=0x12, n=n, seed=9)
    assert cnt.sum() == n and np.array_equal(np.bincount(z, minlength=16), cnt)
    sd = np.sqrt(n * P * (1 - P))
    assert np.all(np.abs(cnt - n * P) <= 5 * sd + 1)
    anc = np.zeros(16)
    for j in range(n):
        anc[m.ancestral_sample(b, a, [j, 0x12, 0, 7], [9, 0])] += 1
    tv = 0.5 * np.abs(anc / n - cnt / n).sum()
    assert tv < 0.015


def test_draw_keying_follows_appendix_a():
    gm = W.random_map(6, 6, 0.2, seed=8)
    m = O.Model.grid(gm, acc=0.9)
    b = W.uniform_belief(gm)
    qpath = 0x0000_0001_0000_0003
    P, R, z, flag, cnt = m.qnode_sample(b, 2, qpath=qpath, n=16, seed=77, step=5, episode=3)
    for j in range(16):
        w = O.philox([j, qpath & 0xFFFFFFFF, qpath >> 32, 5], [77, 3])
        k, f = O.inverse_cdf(P, O.uniform(w[0]))
        assert z[j] == k and flag[j] == f


# ---- P12 / P15 backup recompute and determinism ---------------------------------------------
def test_backup_recompute_bit_exact_and_determinism():
    gm = W.CONFIGS["C1"]["map"]()
    m = O.Model.grid(gm, action_mask=W.A4)
    _, _, Q, _, _ = m.value_iteration(1e-9)
    b = W.uniform_belief(gm)
    r = m.plan(Q, b, depth=2, n=4, seed=1, trace=True, capture_beliefs=True)
    r2 = m.plan(Q, b, depth=2, n=4, seed=1, trace=True, capture_beliefs=True)
    assert np.array_equal(r.qroot, r2.qroot)
    assert np.array_equal(r.trace.q_Q, r2.trace.q_Q) and np.array_equal(r.trace.q_z, r2.trace.q_z)
    t = r.trace
    vval = {int(p): v for p, v in zip(t.v_path, t.v_V)}
    qval = {(int(p), int(l)): q for p, l, q in zip(t.q_path, t.q_level, t.q_Q)}
    n = 4
    for i in range(len(t.q_path)):
        p, lvl = int(t.q_path[i]), int(t.q_level[i])
        acc = 0.0
        for z in range(16):
            c = int(t.q_cnt[i, z])
            if c:
                acc += (c / n) * vval[O.vpath_child(p, lvl, z)]
        assert t.q_R[i] + 0.95 * acc == t.q_Q[i]
    for i in range(len(t.v_path)):
        p, lvl = int(t.v_path[i]), int(t.v_level[i])
        if lvl < 2:
            kids = [qval[(O.qpath_child(p, lvl, a), lvl)] for a in m.action_ids]
            assert max(kids) == t.v_V[i]
    # root Q-nodes
    roots = [qval[(O.qpath_child(0, 0, a), 0)] for a in m.action_ids]
    assert np.array_equal(np.array(roots), r.qroot)
    # the tree is 12 / ~123 V-nodes at C1 (SURVEY §8.0 sizing)
    assert 8 <= (t.v_level == 1).sum() <= 16


# ---- P13 symmetry ---------------------------------------------------------------------------
def test_mirror_symmetry_exact():
    gm = W.from_ascii("""
#...#
..#..
.....
..G..
""")
    m = O.Model.grid(gm, action_mask=W.A9, acc=0.9)
    _, _, Q, _, _ = m.value_iteration(1e-10)
    b = W.uniform_belief(gm)
    r = m.plan(Q, b, depth=2, n=4, mode=O.MODE_BRUTE)
    q = dict(zip(m.action_ids, r.qroot))
    for a, ma in ((0, 2), (3, 5), (6, 8)):
        assert q[a] == pytest.approx(q[ma], abs=1e-12)


# ---- P10 / P14 episodes -----------------------------------------------------------------------
def _bfs_dist(gm, start, diag=True):
    H, Wd = gm.height, gm.width
    dist = {start: 0}
    dq = deque([start])
    moves = [(dr, dc) for dr in (-1, 0, 1) for dc in (-1, 0, 1) if (dr, dc) != (0, 0)
             and (diag or dr == 0 or dc == 0)]
    while dq:
        x = dq.popleft()
        r, c = divmod(x, Wd)
        for dr, dc in moves:
            rr, cc = r + dr, c + dc
            if 0 <= rr < H and 0 <= cc < Wd and gm.occupancy[rr * Wd + cc] == 0:
                y = rr * Wd + cc
                if y not in dist:
                    dist[y] = dist[x] + 1
                    dq.append(y)
    return dist


@pytest.mark.parametrize("planner", [O.PLANNER_QVTS, O.PLANNER_MDP, O.PLANNER_ASTAR])
def test_noise_free_episode_length_equals_bfs(planner):
    gm = W.random_map(9, 10, 0.2, seed=11)
    m = O.Model.grid(gm, action_mask=W.A9, p_int=1.0, p_stay=0.0, p_lat=0.0, acc=1.0)
    _, _, Q, _, _ = m.value_iteration(1e-10)
    dist = _bfs_dist(gm, gm.goal)
    for s in range(3):
        start = W.free_cell(gm, 100 + s)
        rec, la, lz, lx = m.run_episode(Q, W.point_belief(gm, start), planner, depth=2, n=4,
                                        max_steps=200, seed=5, episode=s)
        assert rec.outcome == 0 and rec.collisions == 0
        assert rec.steps == dist[start] + 3
        assert m.astar_length(start) == dist[start]


def test_episode_bookkeeping_replay():
    gm = W.random_map(8, 8, 0.2, seed=12)
    m = O.Model.grid(gm, action_mask=W.A9, acc=0.9)
    _, _, Q, _, _ = m.value_iteration(1e-10)
    b0 = W.uniform_belief(gm)
    rec, la, lz, lx = m.run_episode(Q, b0, O.PLANNER_MDP, max_steps=60, seed=3, episode=2)
    b = b0.copy()
    x = rec.x0
    ret, disc = 0.0, 1.0
    for s in range(rec.steps):
        a_idx = m.action_ids.index(int(la[s]))
        mode = m.belief_mode(b)
        assert m.action_ids[int(np.argmax(Q[:, mode]))] == la[s]     # MDP on the replayed belief
        ret += disc * m.R(x, a_idx)
        disc *= 0.95
        b, _ = m.belief_update(b, a_idx, int(lz[s]))
        x = int(lx[s])
    assert ret == pytest.approx(rec.disc_return, abs=1e-12)
    assert x == rec.x_final


# ---- FIB (Eq. 6-7, NEXT-1) ----------------------------------------------------------------------
def test_fib_identity_observation_equals_mdp():
    """O = identity (|Z| = |X|): FIB is the MDP Q-function."""
    rng = np.random.default_rng(3)
    nx, na = 6, 3
    T = rng.random((nx, na, nx)) ** 3
    T /= T.sum(axis=2, keepdims=True)
    R = -rng.random((nx, na))
    m = O.Model.dense(T, np.eye(nx), R, 0.9)
    st, alpha, it, res = m.fib(1e-11)
    st2, V, Q, _, _ = m.value_iteration(1e-11)
    assert st == O.OK and st2 == O.OK
    assert np.allclose(alpha, Q, atol=1e-9)


def test_fib_uninformative_observation_closed_form():
    """Uniform O: the z-sum collapses, alpha^a = R(.,a) + gamma max_a' T_a alpha^a' (one a' per
    (x,a)) — iterated here with dense matrices."""
    rng = np.random.default_rng(5)
    nx, na, nz = 5, 3, 4
    T = rng.random((nx, na, nx))
    T /= T.sum(axis=2, keepdims=True)
    R = -rng.random((nx, na))
    m = O.Model.dense(T, np.full((nx, nz), 1.0 / nz), R, 0.85)
    st, alpha, _, _ = m.fib(1e-12)
    a = np.full((na, nx), R.max() / (1 - 0.85))
    for _ in range(2000):
        nxt = np.stack([R[:, k] + 0.85 * np.max(np.stack([T[:, k, :] @ a[k2] for k2 in range(na)]), axis=0)
                        for k in range(na)])
        if np.max(np.abs(nxt - a)) < 1e-13:
            a = nxt
            break
        a = nxt
    assert np.allclose(alpha, a, atol=1e-10)


def test_fib_constant_reward_and_bounds_on_grid():
    T = np.zeros((3, 2, 3))
    for i in range(3):
        T[i, 0, i] = 1
        T[i, 1, (i + 1) % 3] = 1
    m = O.Model.dense(T, np.array([[0.7, 0.3], [0.2, 0.8], [0.5, 0.5]]), np.full((3, 2), -2.0), 0.8)
    st, alpha, _, _ = m.fib(1e-12)
    assert np.allclose(alpha, -2.0 / 0.2, atol=1e-9)
    gm = W.random_map(9, 10, 0.2, seed=13)
    g = O.Model.grid(gm, action_mask=W.A8, acc=0.9)
    st, alpha, it, res = g.fib(1e-9)
    _, V, Q, _, _ = g.value_iteration(1e-9)
    free = gm.occupancy == 0
    assert st == O.OK and res < 1e-9
    # FIB is an upper bound no looser than Q_MDP (the max over a' moved inside the z-sum)
    assert np.all(alpha[:, free] <= Q[:, free] + 1e-9)
    assert np.any(alpha[:, free] < Q[:, free] - 1e-3)


# ---- NEXT-3: Alg. 4 literal (ancestral) sampler inside the plan ------------------------------
def test_ancestral_sampler_in_plan_matches_alg4_and_marginal():
    gm = W.random_map(8, 9, 0.2, seed=4)
    m = O.Model.grid(gm, action_mask=W.A8, acc=0.85)
    b = W.random_belief(gm, 6)
    qpath = 0x27
    P, R, z, flag, cnt = m.qnode_sample(b, 3, qpath, 40000, seed=5, step=2, sampler=O.SAMPLER_ANCESTRAL)
    for j in range(0, 40000, 997):   # each draw is Alg. 4 on Philox words 1..3 of its counter
        assert z[j] == m.ancestral_sample(b, 3, [j, qpath, 0, 2], [5, 0])
    n = 40000
    sd = np.sqrt(n * P * (1 - P))
    assert np.all(np.abs(cnt - n * P) <= 5 * sd + 1)      # distribution = the marginal P(z|b,a)


# ---- NEXT-2 (part A): PBVI lower bound (§IV-B) --------------------------------------------------
def _chain(nx=5, gamma=0.9, left_cost=-1.0):
    """Deterministic left/right chain, perfectly observed (O = identity), goal at the right end."""
    T = np.zeros((nx, 2, nx))
    R = np.full((nx, 2), -1.0)
    R[:, 0] = left_cost
    for x in range(nx):
        T[x, 0, max(0, x - 1)] = 1
        T[x, 1, min(nx - 1, x + 1)] = 1
    R[nx - 1, :] = 0.0
    return O.Model.dense(T, np.eye(nx), R, gamma)


def test_pbvi_zero_sweeps_is_the_blind_bound():
    gm = W.random_map(6, 7, 0.2, seed=2)
    m = O.Model.grid(gm, action_mask=W.A8, acc=0.9)
    b0 = W.uniform_belief(gm)
    pts, al, _ = m.pbvi(b0, expansions=2, max_points=8, seed=1, sweeps=0)
    rmin = min(m.R(x, a) for x in range(m.nx) for a in range(m.na) if gm.occupancy[x] == 0)
    for b in pts:
        assert max(a @ b for a in al) == pytest.approx(rmin / (1 - 0.95), abs=1e-12)


def _flagged_qnode(m, b, sampler, n=60000):
    """First Q-node (over tree paths 1, 2, ...) with a flagged draw among n samples."""
    for qpath in range(1, 400):
        P, R, z, flag, cnt = m.qnode_sample(b, qpath % m.na, qpath, n, seed=2, sampler=sampler)
        if flag.any():
            return qpath, P, z, flag
    raise AssertionError("no flagged draw found")


def test_replay_takes_only_a_category_at_the_flagged_boundary():
    """SURVEY c.5 step 3 / reading R11: where the oracle flags a draw (u C_15 within 1e-6 of a CDF
    boundary) it follows the GPU's category only if that category borders the near boundary; a
    far category, or any replay of a non-flagged draw, is ignored."""
    gm = W.random_map(12, 12, 0.2, seed=3)
    m = O.Model.grid(gm, action_mask=W.A8)
    b = W.random_belief(gm, 4)
    n = 60000
    qpath, P, z, flag = _flagged_qnode(m, b, 0, n)
    a = qpath % m.na
    j = int(np.flatnonzero(flag)[0])
    zo = int(z[j])
    live = [k for k in range(16) if P[k] > 0]
    lower = max([k for k in live if k < zo], default=None)
    upper = min([k for k in live if k > zo], default=None)
    far = [k for k in live if k not in (lower, zo, upper)]
    for f in far[:3]:
        _, _, z2, _, _ = m.qnode_sample(b, a, qpath, n, seed=2, replay=[(qpath, j, f)])
        assert np.array_equal(z2, z)
    took = 0
    for cand in (lower, upper):
        if cand is None:
            continue
        _, _, z3, _, _ = m.qnode_sample(b, a, qpath, n, seed=2, replay=[(qpath, j, cand)])
        assert np.array_equal(np.delete(z3, j), np.delete(z, j))
        took += int(z3[j] == cand)
    assert took == 1                     # exactly the neighbour across the near boundary
    j2 = int(np.flatnonzero(~flag)[0])
    _, _, z4, _, _ = m.qnode_sample(b, a, qpath, n, seed=2, replay=[(qpath, j2, (int(z[j2]) + 1) % 16)])
    assert np.array_equal(z4, z)


def test_ancestral_replay_ignores_a_state_off_the_flagged_boundary():
    """The same rule for Alg. 4's state draw (NEXT-3): a replayed state index x is taken only if
    it borders the flagged boundary of the state CDF; cells far from it change nothing."""
    gm = W.random_map(12, 12, 0.2, seed=3)
    m = O.Model.grid(gm, action_mask=W.A8)
    b = W.random_belief(gm, 4)
    n = 2000
    qpath, P, z, flag = _flagged_qnode(m, b, 1, n)
    a = qpath % m.na
    j = int(np.flatnonzero(flag)[0])
    free = np.flatnonzero(gm.occupancy == 0)
    for x in list(free[::17][:6]) + [int(np.flatnonzero(gm.occupancy)[0])]:
        _, _, z2, _, _ = m.qnode_sample(b, a, qpath, n, seed=2, sampler=1, replay=[(qpath, j, 0, int(x))])
        assert np.array_equal(z2, z), x


def test_pbvi_expansion_takes_the_farthest_candidate():
    """PAPER.md:126 (§IV-B): a new belief point is generated from a point already in the set by
    forward sampling, keeping the candidate farthest (L1) from the set.  Hand-built case where the
    farthest, the nearest and the first candidate differ: noise-free motion (p_int = 1), perfect
    sensing, a 9x9 open room, b0 a 2x2 block (a, b / c, d) = (0.3, 0.1 / 0.45, 0.15) in the interior
    where every cell has wall signature 0 -- so each of the 8 moves gives one posterior, b0
    shifted.  L1 distances to b0 (derived by hand): a shift by a diagonal with the overlapping pair
    (a, d) or (b, c) gives 2 - 2 min of the pair, an axis shift 1 + the two differences across it:
    up-left/down-right 1.7, up/down 1.2, up-right/down-left 1.8, left/right 1.5.  Farthest =
    up-right (ties to the lowest stencil id, reading B4); first = up-left; nearest = up."""
    gm = W.from_ascii("\n".join(["." * 9] * 4 + ["....G...."] + ["." * 9] * 4))
    m = O.Model.grid(gm, action_mask=W.A8, p_int=1.0, p_stay=0.0, p_lat=0.0, acc=1.0)
    b0 = np.zeros(81)
    for (r, c), w in {(3, 3): 0.3, (3, 4): 0.1, (4, 3): 0.45, (4, 4): 0.15}.items():
        b0[r * 9 + c] = w
    pts, _, _ = m.pbvi(b0, expansions=1, max_points=2, seed=5, sweeps=0)
    assert pts.shape[0] == 2
    want = np.zeros(81)                       # b0 moved up-right: (r, c) -> (r - 1, c + 1)
    for (r, c), w in {(3, 3): 0.3, (3, 4): 0.1, (4, 3): 0.45, (4, 4): 0.15}.items():
        want[(r - 1) * 9 + c + 1] = w
    assert np.max(np.abs(pts[1] - want)) <= 1e-15
    assert np.sum(np.abs(pts[1] - b0)) == pytest.approx(1.8, abs=1e-12)


def test_pbvi_perfect_observation_chain_reaches_mdp_values():
    m = _chain()
    b0 = np.eye(5)[0]
    pts, al, _ = m.pbvi(b0, expansions=6, max_points=8, seed=3, sweeps=400)
    _, V, Q, _, _ = m.value_iteration(1e-12)
    for b in pts:                      # the expansion reaches point masses along the chain
        x = int(np.argmax(b))
        assert b[x] == 1.0
        assert max(a @ b for a in al) == pytest.approx(V[x], abs=1e-9)


def test_pbvi_backup_uses_the_chosen_actions_reward():
    """Action-dependent rewards on the perfectly observed chain (left costs -2): PBVI's point
    backups still reach V*(x) at the point masses, which requires R(., a*) of the chosen a*."""
    m = _chain(left_cost=-2.0)
    b0 = np.eye(5)[0]
    pts, al, act = m.pbvi(b0, expansions=6, max_points=8, seed=3, sweeps=400)
    _, V, Q, _, _ = m.value_iteration(1e-12)
    for b in pts:
        x = int(np.argmax(b))
        assert max(a @ b for a in al) == pytest.approx(V[x], abs=1e-9)
    for b, a in zip(pts, act):                    # moving right is optimal everywhere but the goal
        if int(np.argmax(b)) != 4:
            assert a == 1


def test_pbvi_sandwich_and_monotone_sweeps():
    gm = W.random_map(6, 8, 0.2, seed=6)
    m = O.Model.grid(gm, action_mask=W.A8, acc=0.85)
    b0 = W.uniform_belief(gm)
    _, A, _, _ = m.fib(1e-9)
    prev = None
    for sw in (5, 10, 20):
        pts, al, _ = m.pbvi(b0, expansions=3, max_points=8, seed=2, sweeps=sw)
        vals = np.array([max(a @ b for a in al) for b in pts])
        probes = list(pts) + [W.random_belief(gm, s) for s in range(4)]
        for b in probes:               # V_PBVI <= V_FIB (<= Q_MDP)
            assert max(a @ b for a in al) <= max(A @ b) + 1e-9
        if prev is not None:           # from the blind lower bound, values at B never decrease
            assert np.all(vals >= prev - 1e-12)
        prev = vals


# ---- anytime best-first QVTS (Alg. 1-7, Eq. 8) ----------------------------
def test_bf_update_rules_spec_examples():
    """SPEC.md:340-350 hand values: Alg. 7 keeps H of the argmax-U child (not the larger H);
    Alg. 6 weights 0.55/0.45 with gaps 2/1 give H_Q = 0.95 max(1.10, 0.45) = 1.045."""
    U, L, H, E = O.bf_v_update([5.0, 3.0], [1.0, 2.0], [2.0, 4.0], [10, 11])
    assert (U, L, H, E) == (5.0, 2.0, 2.0, 10)
    assert O.bf_v_update([1.0, 1.0], [0.0, 0.0], [3.0, 3.0], [7, 8])[3] == 7       # ties -> first
    UQ, LQ, HQ, EQ = O.bf_q_update(-1.0, 0.95, [0.55, 0.45], [0.0, 0.0], [-2.0, -1.0], [2.0, 1.0], [3, 4])
    assert HQ == pytest.approx(1.045, abs=1e-15) and EQ == 3
    assert LQ == pytest.approx(-1.0 + 0.95 * (0.55 * -2.0 + 0.45 * -1.0), abs=1e-15)
    UQ, _, _, _ = O.bf_q_update(-1.0, 0.95, [1.0], [-3.0], [-4.0], [1.0], [0])       # single child
    assert UQ == pytest.approx(-1.0 + 0.95 * -3.0, abs=1e-15)


def _bounds(m, gm, b0, sweeps=20):
    _, A, _, _ = m.fib(1e-9)
    pts, al, act = m.pbvi(b0, expansions=3, max_points=8, seed=2, sweeps=sweeps)
    return A, al, act


def test_bf_zero_expansions_is_the_leaf():
    gm = W.random_map(6, 7, 0.2, seed=3)
    m = O.Model.grid(gm, action_mask=W.A8, acc=0.9)
    b0 = W.random_belief(gm, 2)
    A, al, act = _bounds(m, gm, b0)
    r = m.best_first(A, al, act, b0, n=8, expansions=0)
    assert r["n_exp"] == 0 and r["stop"] == 0
    assert r["U"] == pytest.approx(max(A @ b0), abs=1e-12)
    assert r["L"] == pytest.approx(max(al @ b0), abs=1e-12)
    assert r["action"] == act[int(np.argmax(al @ b0))]


def test_bf_one_expansion_matches_depth1_plan_with_fib_leaves():
    """One expansion with terminal children is a depth-1 tree: U_Q(a) is or_plan's Q(root, a)
    with the FIB alpha-vectors as leaf vectors (same Philox keys), and in EXACT mode
    L_Q(a) = R(b,a) + gamma sum_z P(z|b,a) V_PBVI(Phi(b,a,z)) (Eq. 2)."""
    gm = W.random_map(7, 6, 0.2, seed=5)
    m = O.Model.grid(gm, action_mask=W.A8, acc=0.9)
    b0 = W.random_belief(gm, 4)
    A, al, act = _bounds(m, gm, b0)
    r = m.best_first(A, al, act, b0, n=16, expansions=1, max_depth=1, seed=3, step=2)
    p = m.plan(A, b0, 1, 16, seed=3, step=2)
    assert r["n_exp"] == 1 and r["stop"] == 0
    assert np.max(np.abs(r["UQ"] - p.qroot)) <= 1e-12
    r = m.best_first(A, al, act, b0, n=16, expansions=1, max_depth=1, mode=O.MODE_EXACT)
    for a in range(m.na):
        bbar = m.predict(b0, a)
        P = m.marginal(bbar)
        acc = 0.0
        for z in range(16):
            if P[z] > 1e-300:
                bz, _ = m.belief_update(b0, a, z)
                acc += P[z] * max(al @ bz)
        assert r["LQ"][a] == pytest.approx(m.belief_reward(b0, a) + 0.95 * acc, abs=1e-12)


def test_bf_exact_weights_bounds_tighten_monotonically():
    """With exact weights each expansion replaces a leaf interval by a Bellman image of its
    children's intervals; FIB and PBVI are uniformly improvable (V_PBVI <= H V_PBVI,
    H V_FIB <= V_FIB), so the root U never rises and L never falls (Sec. IV-C anytime)."""
    gm = W.random_map(6, 7, 0.2, seed=8)
    m = O.Model.grid(gm, action_mask=W.A8, acc=0.9)
    b0 = W.uniform_belief(gm)
    A, al, act = _bounds(m, gm, b0, sweeps=30)
    r = m.best_first(A, al, act, b0, n=1, expansions=25, max_depth=4, mode=O.MODE_EXACT)
    rt = r["root_trace"]
    assert r["n_exp"] >= 5
    assert np.all(np.diff(rt[:, 0]) <= 1e-12) and np.all(np.diff(rt[:, 1]) >= -1e-12)
    assert np.all(rt[:, 1] <= rt[:, 0] + 1e-9)
    assert rt[-1, 0] - rt[-1, 1] < rt[0, 0] - rt[0, 1]
    v = r["v"]
    assert np.all(v["L"] <= v["U"] + 1e-9)


def test_bf_E_pointer_is_a_leaf_and_H_is_its_discounted_gap():
    """Alg. 6/7 carry H upward as gamma w H of the selected child: root H = prod(gamma w) H(E)
    along the path to E = root.E, and E is an unexpanded V-node."""
    gm = W.random_map(6, 8, 0.2, seed=9)
    m = O.Model.grid(gm, action_mask=W.A8, acc=0.9)
    b0 = W.uniform_belief(gm)
    A, al, act = _bounds(m, gm, b0)
    r = m.best_first(A, al, act, b0, n=8, expansions=12, max_depth=5, seed=4)
    v = r["v"]
    e = int(v["E"][0])
    assert v["expanded"][e] == 0
    path = int(v["path"][e])
    by_path = {int(p): i for i, p in enumerate(v["path"])}
    prod = 1.0
    for lvl in range(int(v["depth"][e])):         # ancestors' children along the path
        sub = path & ((1 << (8 * (lvl + 1))) - 1)
        prod *= 0.95 * v["w"][by_path[sub]]
    assert v["H"][0] == pytest.approx(prod * v["H"][e], rel=1e-12, abs=1e-15)
    assert v["H"][0] >= 0.0


def test_bf_degenerate_bounds_stop_at_once():
    """Identity O: FIB = MDP and PBVI reaches the MDP values at the point masses, so
    the root gap is 0 and planning finishes before any expansion (SPEC new_tree example)."""
    m = _chain()
    b0 = np.eye(5)[0]
    _, A, _, _ = m.fib(1e-12)
    pts, al, act = m.pbvi(b0, expansions=6, max_points=8, seed=3, sweeps=400)
    r = m.best_first(A, al, act, b0, n=4, expansions=10, gap_tol=1e-6)
    assert r["stop"] == 1 and r["n_exp"] == 0


def test_bf_advance_root_reuses_the_subtree():
    """s.update(a, z) (Alg. 1; SPEC advance_root): the sampled child becomes the root with its
    subtree; its belief is Eq. 3's Phi(b0, a, z); kept nodes lose one level (path >> 8, depth - 1);
    root.E stays inside the new subtree; an unsampled z is refused."""
    gm = W.random_map(6, 8, 0.2, seed=9)
    m = O.Model.grid(gm, action_mask=W.A8, acc=0.9)
    b0 = W.uniform_belief(gm)
    A, al, act = _bounds(m, gm, b0)
    t = O.BfTree(m, A, al, act, b0, 8, 15, max_depth=6, seed=4)
    r0 = t.result()
    v0 = r0["v"]
    a_id = r0["action"]
    j = m.action_ids.index(a_id)
    kids = [i for i in range(r0["n_v"]) if v0["depth"][i] == 1 and (int(v0["path"][i]) & 15) == a_id + 1]
    assert kids
    c = kids[0]
    z = int(v0["path"][c]) >> 4 & 15
    unsampled = [zz for zz in range(16) if all((int(v0["path"][i]) >> 4 & 15) != zz for i in kids)]
    sub_old = {int(v0["path"][i]): i for i in range(r0["n_v"])
               if v0["depth"][i] >= 1 and (int(v0["path"][i]) & 0xFF) == (int(v0["path"][c]) & 0xFF)}
    assert t.advance(a_id, z)
    r1 = t.cont(8, 0, max_depth=6, seed=4, step=1)
    assert r1["root"] == c and r1["U"] == v0["U"][c] and r1["L"] == v0["L"][c]
    bz, _ = m.belief_update(b0, j, z)
    assert np.max(np.abs(t.belief(c) - bz)) <= 1e-15
    v1 = r1["v"]
    alive = [i for i in range(r1["n_v"]) if v1["depth"][i] >= 0]
    assert sorted(alive) == sorted(sub_old.values())
    for p_old, i in sub_old.items():
        assert int(v1["path"][i]) == p_old >> 8 and v1["depth"][i] == v0["depth"][i] - 1
    assert v1["depth"][int(v1["E"][c])] >= 0                 # root.E inside the kept subtree
    r2 = t.cont(8, 10, max_depth=6, seed=4, step=1)
    assert r2["n_exp"] > 0 and r2["root"] == c
    if unsampled:
        t2 = O.BfTree(m, A, al, act, b0, 8, 15, max_depth=6, seed=4)
        assert not t2.advance(a_id, unsampled[0])
        t2.close()
    t.close()
