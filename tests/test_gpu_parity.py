"""GPU parity: the CUDA path (through the C ABI) against the fp64 oracle, element by element on
the same seeded inputs.  Run on a B200 with `pytest -m gpu`."""
import numpy as np
import pytest

import oracle as O
import workloads as W
from tests import parity as PT

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def Q():
    assert torch.cuda.is_available(), "GPU tests need CUDA"
    from paper_1810_00204_b200 import qvts
    qvts.lib()
    return qvts


def pair(Q, gm, mask, acc=0.95, p=(0.8, 0.1, 0.05)):
    gmod = Q.Model(gm, action_mask=mask, p_intended=p[0], p_stay=p[1], p_lateral=p[2], sensor_acc=acc)
    code, sweeps, res = gmod.value_iteration(1e-9)
    assert code == 0 and res < 1e-9
    omod = O.Model.grid(gm, action_mask=mask, p_int=p[0], p_stay=p[1], p_lat=p[2], acc=acc)
    st, V, Qo, osw, ores = omod.value_iteration(1e-9)
    assert st == O.OK
    return gmod, omod, Qo, sweeps, osw


def dev(b):
    return torch.tensor(np.asarray(b, np.float32), device="cuda")


MAPS = {
    "C1": (lambda: W.CONFIGS["C1"]["map"](), W.A4),
    "ragged": (lambda: W.random_map(29, 37, 0.2, seed=9), W.A8),
    "paper": (lambda: W.paper_style(50, 50, 6, 12, seed=1), W.A9),
}


@pytest.mark.parametrize("name", list(MAPS))
def test_tables_and_value_iteration(Q, name):
    gm, mask = MAPS[name][0](), MAPS[name][1]
    g, o, Qo, sweeps, osw = pair(Q, gm, mask)
    R, sig = g.tables()
    assert np.array_equal(sig, o.sig_table().astype(np.uint8))
    assert np.max(np.abs(R.astype(np.float64) - o.R_table())) <= 2.5e-7
    assert abs(sweeps - osw) <= 1
    assert np.max(np.abs(g.q() - Qo)) <= 1e-7


@pytest.mark.parametrize("name", list(MAPS))
def test_belief_update(Q, name):
    gm, mask = MAPS[name][0](), MAPS[name][1]
    g, o, _, _, _ = pair(Q, gm, mask)
    for seed in (1, 2):
        b = W.random_belief(gm, seed, sparsity=0.3 if seed == 2 else 0.0)
        bd = dev(b)
        b32 = np.asarray(b, np.float32).astype(np.float64)
        out = torch.empty_like(bd)
        for a in g.action_ids:
            ai = o.action_ids.index(a)
            for z in (0, 3, 5, 15):
                ref, pref = o.belief_update(b32, ai, z)
                p = g.belief_update(bd, a, z, out)
                assert abs(p - pref) <= 1e-7, (a, z, p, pref)
                got = out.cpu().numpy().astype(np.float64)
                assert np.max(np.abs(got - ref)) <= PT.TOL
                assert np.max(np.abs(got - ref)) <= 1e-5 * max(1e-3, ref.max())
                assert np.all(got[gm.occupancy == 1] == 0.0)


def test_belief_update_zero_likelihood(Q):
    gm = W.pillars(6, 6, 1, seed=3)
    g = Q.Model(gm, action_mask=W.A9, sensor_acc=1.0)
    g.value_iteration()
    b = dev(W.point_belief(gm, W.free_cell(gm, 1)))
    out = torch.empty_like(b)
    o = O.Model.grid(gm, action_mask=W.A9, acc=1.0)
    P = o.marginal(o.predict(np.asarray(b.cpu(), np.float64), 4))
    z = int(np.flatnonzero(P == 0)[0])
    with pytest.raises(Q.QvtsError) as e:
        g.belief_update(b, 4, z, out)
    assert e.value.code == 5


def run_parity(Q, gm, mask, depth, n, b0, seed=1, step=0, episode=0, beliefs=True, sampler=0):
    g, o, Qo, _, _ = pair(Q, gm, mask)
    b32 = np.asarray(b0, np.float32)
    res = g.plan_step(dev(b32), depth, n, seed=seed, step=step, episode=episode, want_trace=True, sampler=sampler)
    gq, gv, gbel, _ = PT.gpu_tree(g, n, with_beliefs=beliefs, with_states=(sampler == Q.QVTS_SAMPLER_ANCESTRAL))
    ores = o.plan(Qo, b32.astype(np.float64), depth, n, seed=seed, step=step, episode=episode, trace=True,
                  capture_beliefs=beliefs, sampler=sampler)
    oq, ov, obel = PT.oracle_tree(ores)
    replay, nmis = PT.draw_mismatches(gq, oq)
    if replay:   # flagged draws decided differently: replay the GPU's decision in the oracle
        ores = o.plan(Qo, b32.astype(np.float64), depth, n, seed=seed, step=step, episode=episode, trace=True,
                      capture_beliefs=beliefs, replay=replay, sampler=sampler)
        oq, ov, obel = PT.oracle_tree(ores)
        PT.draw_mismatches(gq, oq)
    err = PT.compare_trees(gq, gv, oq, ov, gbel if beliefs else None, obel if beliefs else None)
    assert np.max(np.abs(np.array(res.q_root[:g.n_actions]) - ores.qroot)) <= PT.TOL
    PT.check_action(res.action, ores.action, ores.qroot, g.action_ids)
    assert res.n_belief_updates == len(ov)
    return res, err, nmis


def test_plan_C1_full_tree(Q):
    gm = W.CONFIGS["C1"]["map"]()
    res, err, _ = run_parity(Q, gm, W.A4, 2, 4, W.uniform_belief(gm))
    assert res.n_vnodes[1] >= 8


@pytest.mark.parametrize("seed,step", [(1, 0), (7, 3)])
def test_plan_ragged_depth3(Q, seed, step):
    gm = W.random_map(29, 37, 0.2, seed=9)
    run_parity(Q, gm, W.A8, 3, 8, W.random_belief(gm, 5), seed=seed, step=step, episode=2)


def test_plan_paper_style_A9(Q):
    gm = W.paper_style(50, 50, 6, 12, seed=1)
    run_parity(Q, gm, W.A9, 3, 16, W.uniform_belief(gm), beliefs=False)


def test_plan_depth1_and_large_n(Q):
    gm = W.random_map(13, 11, 0.2, seed=2)
    run_parity(Q, gm, W.A9, 1, 300, W.random_belief(gm, 3))
    run_parity(Q, gm, W.A4, 4, 2, W.uniform_belief(gm))


def test_plan_C3_full(Q):
    gm = W.CONFIGS["C3"]["map"]()
    res, err, nmis = run_parity(Q, gm, W.A8, 3, 8, W.uniform_belief(gm), beliefs=False)
    assert res.n_belief_updates > 10000


def test_plan_deterministic(Q):
    gm = W.random_map(40, 40, 0.2, seed=4)
    g, _, _, _, _ = pair(Q, gm, W.A8)
    b = dev(W.uniform_belief(gm, np.float32))
    r1 = g.plan_step(b, 3, 8, seed=3, want_trace=True)
    t1 = g.trace(with_draws=True, n_samples=8)
    r2 = g.plan_step(b, 3, 8, seed=3, want_trace=True)
    t2 = g.trace(with_draws=True, n_samples=8)
    assert list(r1.q_root) == list(r2.q_root)
    for d in range(3):
        for k in ("R", "P", "Q", "z", "cnt"):
            assert np.array_equal(t1["levels"][d]["q"][k], t2["levels"][d]["q"][k])
    assert np.array_equal(t1["leafV"], t2["leafV"])


@pytest.mark.parametrize("G", [2, 3, 4, 8])
def test_sharded_plan_matches_single_gpu_bitwise(Q, G):
    """Run the G ranks of a sharded plan step serially on one GPU: first pass collects each rank's
    zero-padded shard-level values, second pass feeds back their exact sum."""
    gm = W.random_map(40, 44, 0.2, seed=6)
    g, _, _, _, _ = pair(Q, gm, W.A8)
    b = dev(W.uniform_belief(gm, np.float32))
    ref = g.plan_step(b, 3, 8, seed=5)
    partials = {}

    def collect(r):
        def fn(ptr, count, stream):
            t = torch.as_tensor(Q._CudaArray(ptr, count), device="cuda")
            partials[r] = t.cpu().numpy().copy()
        return fn

    for r in range(G):
        g.plan_step(b, 3, 8, seed=5, comm=Q.make_callback_comm(r, G, collect(r), min_nodes_per_rank=4))
    total = sum(partials[r] for r in range(G))
    for r in range(G):
        assert np.count_nonzero(partials[r]) > 0
    nz = [set(np.flatnonzero(partials[r])) for r in range(G)]
    for r in range(G):
        for s in range(r + 1, G):
            assert not (nz[r] & nz[s])    # disjoint ownership

    def feed(ptr, count, stream):
        t = torch.as_tensor(Q._CudaArray(ptr, count), device="cuda")
        t.copy_(torch.from_numpy(total).cuda())

    for r in range(G):
        res = g.plan_step(b, 3, 8, seed=5, comm=Q.make_callback_comm(r, G, feed, min_nodes_per_rank=4))
        assert list(res.q_root) == list(ref.q_root)
        assert res.action == ref.action


def test_C4_full_size_sampled_parity(Q):
    """BASELINE config 4 (256x256, A8, depth 4, n = 16), launched as bench.py times it: sampled
    nodes on every level recomputed one by one by the oracle along their own paths."""
    cfg = W.CONFIGS["C4"]
    gm = cfg["map"]()
    g, o, Qo, _, _ = pair(Q, gm, W.A8)
    b32 = W.uniform_belief(gm, np.float32)
    D, n = cfg["depth"], cfg["n"]
    res = g.plan_step(dev(b32), D, n, seed=1, want_trace=True)
    assert res.n_belief_updates > 1_000_000
    na = g.n_actions
    rng = np.random.default_rng(0)
    # level-0 Q-nodes: exact
    lq0 = Q.qvts_trace_qnodes(g.h, 0, na, n, True)
    b = b32.astype(np.float64)
    for ai, a in enumerate(g.action_ids):
        P, R, z, flag, cnt = o.qnode_sample(b, ai, O.qpath_child(0, 0, a), n, seed=1)
        assert abs(lq0["R"][ai] - R) <= PT.TOL and np.max(np.abs(lq0["P"][ai] - P)) <= 1e-7
        assert np.all((lq0["z"][ai] == z) | flag)
    # random root-to-level-(D-1) paths followed by the oracle
    _, nv, nqw = Q.qvts_trace_counts(g.h)
    vlev = [Q.qvts_trace_vnodes(g.h, d, nv[d]) for d in range(D)]
    qlev = [Q.qvts_trace_qnodes(g.h, d, nqw[d] * na, n, True) for d in range(D)]
    for trial in range(6):
        i = int(rng.integers(nv[D - 1]))
        chain = [i]
        for d in range(D - 1, 0, -1):
            chain.append(int(vlev[d]["parent_q"][chain[-1]]) // na)
        chain = chain[::-1]           # V-node indices at levels 0..D-1
        bo = b32.astype(np.float64)
        for d in range(1, D):
            vi = chain[d]
            qi = int(vlev[d]["parent_q"][vi])
            ai = qi % na
            qpath = int(qlev[d - 1]["path"][qi])
            P, R, z, flag, cnt = o.qnode_sample(bo, ai, qpath, n, seed=1)
            assert abs(qlev[d - 1]["R"][qi] - R) <= PT.TOL
            assert np.max(np.abs(qlev[d - 1]["P"][qi] - P)) <= 1e-6
            mism = qlev[d - 1]["z"][qi] != z
            assert not np.any(mism & ~flag)
            zz = int(vlev[d]["z"][vi])
            assert cnt[zz] > 0 or np.any(mism)
            bo, _ = o.belief_update(bo, ai, zz)
            gb = Q.qvts_trace_belief(g.h, d, vi, g.n_cells).astype(np.float64)
            assert np.max(np.abs(gb - bo)) <= PT.TOL
        # value of the level-(D-1) node with its subtree (its Q-nodes are the leaf Q-level)
        vpath = int(vlev[D - 1]["path"][chain[-1]])
        Vo, qv = o.vnode_value(Qo, bo, vpath, D - 1, D, n, seed=1)
        assert abs(vlev[D - 1]["V"][chain[-1]] - Vo) <= PT.TOL
        w = chain[-1]
        assert np.max(np.abs(qlev[D - 1]["Q"][w * na:(w + 1) * na] - qv)) <= PT.TOL
    # backup identity at the root from the GPU's own arrays (fp64 recompute)
    for d in range(D - 2, -1, -1):
        lq, lc = qlev[d], vlev[d + 1]
        off = np.concatenate([[0], np.cumsum([int((c > 0).sum()) for c in lq["cnt"]])])
        for qi in rng.integers(0, len(lq["R"]), size=min(200, len(lq["R"]))):
            s = sum((lc["f"][c] / n) * lc["V"][c] for c in range(off[qi], off[qi + 1]))
            assert abs(lq["R"][qi] + 0.95 * s - lq["Q"][qi]) <= 1e-9
    assert np.max(np.abs(np.array(res.q_root[:na]) - qlev[0]["Q"])) == 0.0


@pytest.mark.parametrize("name", ["ragged", "paper"])
def test_fib_alpha_and_fib_leaf_plan(Q, name):
    """NEXT-1: FIB alpha-vectors (Eq. 7) against the oracle, then a plan step whose leaves use them."""
    gm, mask = MAPS[name][0](), MAPS[name][1]
    g, o, Qo, _, _ = pair(Q, gm, mask)
    code, sweeps, res = g.fib_iteration(1e-9)
    assert code == 0 and res < 1e-9
    st, Ao, osw, ores = o.fib(1e-9)
    assert st == O.OK and abs(sweeps - osw) <= 1
    A = g.alpha()
    assert np.max(np.abs(A - Ao)) <= 1e-7
    free = gm.occupancy == 0
    assert np.all(A[:, free] <= g.q()[:, free] + 1e-7)          # FIB no looser than Q_MDP
    b32 = np.asarray(W.uniform_belief(gm), np.float32)
    res = g.plan_step(dev(b32), 2, 8, seed=4, want_trace=True, leaf_bound=Q.QVTS_LEAF_FIB)
    gq, gv, _, _ = PT.gpu_tree(g, 8)
    ro = o.plan(Ao, b32.astype(np.float64), 2, 8, seed=4, trace=True)
    oq, ov, _ = PT.oracle_tree(ro)
    replay, _ = PT.draw_mismatches(gq, oq)
    if replay:
        ro = o.plan(Ao, b32.astype(np.float64), 2, 8, seed=4, trace=True, replay=replay)
        oq, ov, _ = PT.oracle_tree(ro)
    PT.compare_trees(gq, gv, oq, ov)
    assert np.max(np.abs(np.array(res.q_root[:g.n_actions]) - ro.qroot)) <= PT.TOL
    PT.check_action(res.action, ro.action, ro.qroot, g.action_ids)


@pytest.mark.parametrize("name,depth,n", [("C1", 2, 4), ("ragged", 3, 8), ("paper", 2, 16)])
def test_plan_ancestral_sampler(Q, name, depth, n):
    """NEXT-3: Alg. 4 literally (x ~ b, x' ~ T, z ~ O on Philox words 1..3) on the GPU."""
    gm, mask = MAPS[name][0](), MAPS[name][1]
    res, err, nmis = run_parity(Q, gm, mask, depth, n, W.random_belief(gm, 8), seed=3, step=1,
                                beliefs=(name != "paper"), sampler=Q.QVTS_SAMPLER_ANCESTRAL)


@pytest.mark.parametrize("name,b0,exp,maxp,sweeps", [("C1", "uniform", 3, 12, 20), ("ragged", "random", 3, 16, 15),
                                                     ("paper", "uniform", 2, 10, 8)])
def test_pbvi_against_oracle(Q, name, b0, exp, maxp, sweeps):
    """NEXT-2: PBVI lower bound — the belief set (Alg. 4 draws + farthest-posterior rule) and the
    alpha-vectors after `sweeps` point-based backups, element by element against the oracle."""
    gm, mask = MAPS[name][0](), MAPS[name][1]
    g = Q.Model(gm, action_mask=mask)
    o = O.Model.grid(gm, action_mask=mask)
    b32 = np.asarray(W.uniform_belief(gm) if b0 == "uniform" else W.random_belief(gm, 5), np.float32)
    pts, al, act = g.pbvi(dev(b32), expansions=exp, max_points=maxp, seed=7, sweeps=sweeps)
    opts, oal, oact = o.pbvi(b32.astype(np.float64), expansions=exp, max_points=maxp, seed=7, sweeps=sweeps)
    assert pts.shape == opts.shape and pts.shape[0] > 1
    assert np.max(np.abs(pts - opts)) <= 1e-12
    assert al.shape == oal.shape
    assert np.max(np.abs(al - oal)) <= 1e-9 * max(1.0, np.max(np.abs(oal)))
    assert np.array_equal(act[:len(oact)], oact)
    # lower bound on the belief points: below FIB's upper bound
    code, _, _ = g.fib_iteration(1e-9)
    A = g.alpha()
    for b in pts:
        assert np.max(al @ b) <= np.max(A @ b) + 1e-9
    g.close()


def test_pbvi_zero_sweeps_and_single_point(Q):
    """Degenerate cases: no sweeps leaves the blind vector; expansions = 0 keeps {b0} only."""
    gm = W.CONFIGS["C1"]["map"]()
    g = Q.Model(gm, action_mask=W.A4)
    pts, al, act = g.pbvi(None, expansions=0, max_points=8, seed=1, sweeps=0)
    assert pts.shape[0] == 1 and al.shape[0] == 1
    o = O.Model.grid(gm, action_mask=W.A4)
    opts, oal, _ = o.pbvi(np.asarray(W.uniform_belief(gm), np.float64), expansions=0, max_points=8, seed=1, sweeps=0)
    assert np.max(np.abs(pts - opts)) <= 1e-15 and np.max(np.abs(al - oal)) == 0.0
    g.close()


def _bf_pair(Q, gm, mask, b32, pbvi_kw):
    g = Q.Model(gm, action_mask=mask)
    o = O.Model.grid(gm, action_mask=mask)
    code, _, _ = g.fib_iteration(1e-9)
    assert code == 0
    g.pbvi(dev(b32), **pbvi_kw)
    st, Ao, _, _ = o.fib(1e-9)
    _, alo, acto = o.pbvi(b32.astype(np.float64), **pbvi_kw)
    return g, o, Ao, alo, acto


@pytest.mark.parametrize("name,n,exps,maxd", [("C1", 8, 25, 4), ("ragged", 16, 30, 5), ("paper", 8, 20, 3)])
def test_best_first_against_oracle(Q, name, n, exps, maxd):
    """NEXT-2: the anytime best-first QVTS (Alg. 1-7, Eq. 8) on the GPU against the oracle: same
    expansion order (near-tied selections replayed, reading B5), every V-node's f, U, L, H, the
    root Q bounds and the executed action."""
    gm, mask = MAPS[name][0](), MAPS[name][1]
    b32 = np.asarray(W.uniform_belief(gm), np.float32)
    g, o, Ao, alo, acto = _bf_pair(Q, gm, mask, b32, dict(expansions=3, max_points=12, seed=5, sweeps=20))
    res = g.plan_best_first(dev(b32), n, exps, max_depth=maxd, seed=2, step=1)
    tr = g.trace_best_first()
    gpaths = tr["path"][tr["exp_order"]]
    r = o.best_first(Ao, alo, acto, b32.astype(np.float64), n, exps, max_depth=maxd, seed=2, step=1,
                     replay=gpaths, replay_tol=1e-4)
    assert r["mism"] == 0
    assert r["subs"] <= max(1, exps // 10)
    assert r["n_exp"] == res.n_expansions and r["stop"] == res.stop_reason
    assert r["n_v"] == res.n_vnodes
    ov = r["v"]
    idx = {int(p): i for i, p in enumerate(ov["path"])}
    scale = max(1.0, float(np.max(np.abs(ov["U"]))))
    for i, p in enumerate(tr["path"]):
        j = idx[int(p)]
        assert tr["f"][i] == ov["f"][j] and tr["depth"][i] == ov["depth"][j]
        assert abs(tr["U"][i] - ov["U"][j]) <= PT.TOL
        assert abs(tr["L"][i] - ov["L"][j]) <= PT.TOL
        assert abs(tr["H"][i] - ov["H"][j]) <= 2 * PT.TOL
        assert bool(tr["expanded"][i]) == bool(ov["expanded"][j])
    assert abs(res.U - r["U"]) <= PT.TOL and abs(res.L - r["L"]) <= PT.TOL
    na = g.n_actions
    assert np.max(np.abs(np.array(res.u_q[:na]) - r["UQ"])) <= PT.TOL
    assert np.max(np.abs(np.array(res.l_q[:na]) - r["LQ"])) <= PT.TOL
    assert np.max(np.abs(tr["root_trace"] - r["root_trace"])) <= PT.TOL
    # executed action: max L_Q (ties by U_Q) -- equal, or the oracle's L_Q values are near-tied
    j = g.action_ids.index(res.action)
    assert res.action == r["action"] or r["LQ"][j] >= np.max(r["LQ"]) - PT.TIE
    g.close()


def test_best_first_stop_rules(Q):
    """planningFinished(): zero budget (root = leaf, PBVI action), a huge gap tolerance, the
    depth cap (terminal E) and the wall-clock budget."""
    gm, mask = MAPS["ragged"][0](), MAPS["ragged"][1]
    b32 = np.asarray(W.random_belief(gm, 3), np.float32)
    g, o, Ao, alo, acto = _bf_pair(Q, gm, mask, b32, dict(expansions=2, max_points=8, seed=1, sweeps=10))
    res = g.plan_best_first(dev(b32), 8, 0)
    r = o.best_first(Ao, alo, acto, b32.astype(np.float64), 8, 0)
    assert res.n_expansions == 0 and res.stop_reason == Q.QVTS_BF_BUDGET and res.action == r["action"]
    assert abs(res.U - r["U"]) <= 1e-5 * abs(r["U"]) and abs(res.L - r["L"]) <= 1e-5 * abs(r["L"])
    res = g.plan_best_first(dev(b32), 8, 50, gap_tol=1e9)
    assert res.n_expansions == 0 and res.stop_reason == Q.QVTS_BF_GAP
    res = g.plan_best_first(dev(b32), 8, 10000, max_depth=1)
    assert res.n_expansions == 1 and res.stop_reason == Q.QVTS_BF_TERMINAL
    import time
    # the budget is checked between chunks of 16 expansions (and before the first, and after a
    # node-pool growth), so a cold call whose setup (pool allocation, graph capture) overruns the
    # budget stops with 0 expansions; warm calls must expand, and stop within the budget plus one
    # chunk or one pool growth with its graph recapture; a growth's allocation time depends on the
    # box (a few hundred ms to ~1 s for a multi-GB pool on a fresh box), hence the loose bound
    g.plan_best_first(dev(b32), 8, 100000, max_depth=8, time_budget_ms=200.0)   # warm: graphs, pool
    for budget in (200.0, 20.0):
        t0 = time.perf_counter()
        res = g.plan_best_first(dev(b32), 8, 100000, max_depth=8, time_budget_ms=budget)
        dt = (time.perf_counter() - t0) * 1e3
        assert res.stop_reason in (Q.QVTS_BF_TIME, Q.QVTS_BF_TERMINAL)
        if res.stop_reason == Q.QVTS_BF_TIME:
            assert dt < budget + 1500.0
            if budget >= 200.0:
                assert res.n_expansions > 0
    g.close()


def _bf_compare(tr, r, scale, alive_only=False):
    ov = r["v"]
    idx = {int(p): i for i, p in enumerate(ov["path"]) if ov["depth"][i] >= 0}
    n = 0
    for i, p in enumerate(tr["path"]):
        if tr["depth"][i] < 0:
            continue
        j = idx[int(p)]
        n += 1
        assert tr["f"][i] == ov["f"][j] and tr["depth"][i] == ov["depth"][j]
        assert abs(tr["U"][i] - ov["U"][j]) <= PT.TOL
        assert abs(tr["L"][i] - ov["L"][j]) <= PT.TOL
        assert abs(tr["H"][i] - ov["H"][j]) <= 2 * PT.TOL
    assert n == len(idx)


def test_best_first_tree_reuse_against_oracle(Q):
    """NEXT-4 (tree reuse): plan, s.update(a, z) keeps the sampled (a, z) subtree with relative
    paths, then more expansions continue it; both trees against the oracle's re-rooted tree."""
    gm, mask = MAPS["ragged"][0](), MAPS["ragged"][1]
    b32 = np.asarray(W.uniform_belief(gm), np.float32)
    g, o, Ao, alo, acto = _bf_pair(Q, gm, mask, b32, dict(expansions=3, max_points=12, seed=5, sweeps=20))
    res1 = g.plan_best_first(dev(b32), 8, 25, max_depth=6, seed=2, step=0)
    tr1 = g.trace_best_first()
    t = O.BfTree(o, Ao, alo, acto, b32.astype(np.float64), 8, 25, max_depth=6, seed=2, step=0,
                 replay=tr1["path"][tr1["exp_order"]])
    r1 = t.result()
    assert r1["mism"] == 0 and r1["n_exp"] == res1.n_expansions
    scale = max(1.0, float(np.max(np.abs(r1["v"]["U"]))))
    _bf_compare(tr1, r1, scale)
    a_id = res1.action
    kids = [i for i in range(len(tr1["path"])) if tr1["depth"][i] == 1 and (int(tr1["path"][i]) & 15) == a_id + 1]
    z = int(tr1["path"][kids[-1]]) >> 4 & 15
    assert g.bf_advance(a_id, z) and t.advance(a_id, z)
    absent = [zz for zz in range(16) if all((int(tr1["path"][i]) >> 4 & 15) != zz for i in kids)]
    res2 = g.plan_best_first(None, 8, 20, max_depth=6, seed=2, step=1, reuse=True)
    tr2 = g.trace_best_first()
    r2 = t.cont(8, 20, max_depth=6, seed=2, step=1, replay=tr2["path"][tr2["exp_order"]])
    assert r2["mism"] == 0 and r2["n_exp"] == res2.n_expansions and r2["stop"] == res2.stop_reason
    _bf_compare(tr2, r2, scale)
    assert abs(res2.U - r2["U"]) <= PT.TOL and abs(res2.L - r2["L"]) <= PT.TOL
    assert np.max(np.abs(tr2["root_trace"] - r2["root_trace"])) <= PT.TOL
    j = g.action_ids.index(res2.action)
    assert res2.action == r2["action"] or r2["LQ"][j] >= np.max(r2["LQ"]) - PT.TIE
    if absent:   # the new root's unsampled z: no reuse
        kids2 = [i for i in range(len(tr2["path"])) if tr2["depth"][i] == 1 and (int(tr2["path"][i]) & 15) == res2.action + 1]
        zs2 = {int(tr2["path"][i]) >> 4 & 15 for i in kids2}
        miss = [zz for zz in range(16) if zz not in zs2]
        if kids2 and miss:
            assert not g.bf_advance(res2.action, miss[0])
    t.close()
    g.close()


# ---- edge shapes and degenerate cases ----------------------------------------------------------
@pytest.mark.parametrize("H,Wd,mask", [(1, 40, W.A8), (3, 203, W.A8), (203, 3, W.A4), (2, 2, W.A9)])
def test_plan_extreme_shapes(Q, H, Wd, mask):
    """One-row, very wide, very tall and 2x2 grids: band construction, halos and clamping at the
    map edge on every side."""
    gm = W.random_map(H, Wd, 0.05, seed=11) if H * Wd > 4 else W.from_ascii("G.\n..")
    run_parity(Q, gm, mask, 2, 4, W.random_belief(gm, 2))


def test_plan_single_free_cell(Q):
    """Every move is blocked: all mass stays, one observation, a one-child chain per action."""
    gm = W.from_ascii("###\n#G#\n###")
    res, _, _ = run_parity(Q, gm, W.A9, 3, 8, W.uniform_belief(gm))
    assert res.n_vnodes[1] >= 9 and res.n_vnodes[3] >= 9 ** 3


def test_plan_depth8_single_draw(Q):
    """The maximum depth (8 action levels, the tree-path limit) with n = 1: 4^8 leaves."""
    gm = W.from_ascii("..#.\n.G..\n#...")
    res, _, _ = run_parity(Q, gm, W.A4, 8, 1, W.uniform_belief(gm), beliefs=False)
    assert res.n_vnodes[8] == 4 ** 8


def test_plan_point_mass_root_and_max_n(Q):
    """A point-mass root in a corner, and the maximum draw count n = 4096 at depth 1."""
    gm = W.random_map(9, 12, 0.15, seed=6)
    b = np.zeros(gm.occupancy.size)
    b[int(np.flatnonzero(gm.occupancy == 0)[0])] = 1.0
    run_parity(Q, gm, W.A8, 3, 8, b)
    run_parity(Q, gm, W.A8, 1, 4096, W.random_belief(gm, 4))


@pytest.mark.parametrize("name", ["C1", "ragged", "paper"])
def test_belief_update_batch(Q, name):
    """Batched Eq. 3 against the oracle element by element, mixed actions and observations."""
    gm, mask = MAPS[name][0](), MAPS[name][1]
    g = Q.Model(gm, action_mask=mask)
    o = O.Model.grid(gm, action_mask=mask)
    rng = np.random.default_rng(3)
    nb = 37
    B = np.stack([W.random_belief(gm, 100 + i) for i in range(nb)]).astype(np.float32)
    acts = rng.choice(g.action_ids, size=nb)
    zs = np.zeros(nb, np.int32)
    for i in range(nb):                     # a z with non-negligible mass
        P = o.marginal(o.predict(B[i].astype(np.float64), g.action_ids.index(acts[i])))
        zs[i] = int(np.argsort(P)[-1 - (i % 3)])
    out = torch.empty((nb, gm.occupancy.size), dtype=torch.float32, device="cuda")
    p = g.belief_update_batch(dev(B), acts, zs, out)
    res = out.cpu().numpy()
    for i in range(nb):
        ob, op = o.belief_update(B[i].astype(np.float64), g.action_ids.index(acts[i]), int(zs[i]))
        assert abs(p[i] - op) <= 1e-7
        assert np.max(np.abs(res[i] - ob)) <= PT.TOL
        assert np.max(np.abs(res[i] - ob)) <= 1e-5 * max(1e-3, float(np.max(ob)))
        assert np.all(res[i][gm.occupancy == 1] == 0.0)
    g.close()


def test_plan_localised_root_skips_tiles(Q):
    """Active-tile skipping (beliefs localise within 20-30 steps,
    PAPER.md:396 §V-B): a localised root on the C3 map (128x128, several row bands per level)
    keeps every belief of a depth-3 tree within 3 cells of the start, so most (parent pair, band)
    tiles hold no mass and are skipped by the hist and leaf kernels (device counter
    n_tiles_skipped > 0); the tree, every belief and every value still match the oracle
    element by element, as does the two-cell root straddling a band boundary."""
    gm = W.CONFIGS["C3"]["map"]()
    free = np.flatnonzero(gm.occupancy == 0)
    near_top = int(free[np.searchsorted(free, 5 * 128 + 40)])
    res, err, _ = run_parity(Q, gm, W.A8, 3, 8, W.point_belief(gm, near_top), seed=3)
    assert res.n_tiles_skipped > 0, res.n_tiles_skipped
    b = np.zeros(gm.occupancy.size)
    for r in (63, 64):                                  # mass on both sides of a band boundary
        row = [x for x in free if r * 128 <= x < (r + 1) * 128]
        b[row[len(row) // 2]] = 0.5
    res2, _, _ = run_parity(Q, gm, W.A8, 3, 8, b, seed=4)
    assert res2.n_tiles_skipped > 0
    # the skip decisions are a function of the beliefs alone: the graph-captured step (no trace)
    # skips the same tiles and returns the same root values bit for bit
    g = Q.Model(gm, action_mask=W.A8)
    g.value_iteration(1e-9)
    rt = g.plan_step(dev(b), 3, 8, seed=4, want_trace=True)
    rg = g.plan_step(dev(b), 3, 8, seed=4)
    assert rt.n_tiles_skipped == rg.n_tiles_skipped == res2.n_tiles_skipped
    assert list(rt.q_root[:g.n_actions]) == list(rg.q_root[:g.n_actions])
    g.close()


@pytest.mark.parametrize("H,Wd", [(200, 256), (37, 64), (256, 16), (64, 1024)])
def test_belief_update_batch_cluster_shapes(Q, H, Wd):
    """The one-pass cluster kernel on the map shapes that change its geometry: 7 CTAs with a short
    last one (200 x 256), one CTA owning every row so both halo rows are off the map (37 x 64),
    64 rows per pass of a 16-wide map (256 x 16), one row per pass and 8 CTAs of 8 rows
    (64 x 1024); A9 (stay included), mixed actions and observations, against the oracle (Eq. 3,
    PAPER.md:59-63) element by element."""
    gm = W.random_map(H, Wd, 0.2, seed=H + Wd)
    g = Q.Model(gm, action_mask=W.A9)
    o = O.Model.grid(gm, action_mask=W.A9)
    rng = np.random.default_rng(H)
    nb = 11
    B = np.stack([W.random_belief(gm, 300 + i, sparsity=0.3 if i % 2 else 0.0) for i in range(nb)]).astype(np.float32)
    acts = np.array([g.action_ids[i % g.n_actions] for i in range(nb)], np.int32)
    rng.shuffle(acts)
    zs = np.zeros(nb, np.int32)
    for i in range(nb):
        P = o.marginal(o.predict(B[i].astype(np.float64), g.action_ids.index(acts[i])))
        zs[i] = int(np.argsort(P)[-1 - (i % 4)])
    out = torch.empty((nb, gm.occupancy.size), dtype=torch.float32, device="cuda")
    p = g.belief_update_batch(dev(B), acts, zs, out)
    res = out.cpu().numpy()
    for i in range(nb):
        ob, op = o.belief_update(B[i].astype(np.float64), g.action_ids.index(acts[i]), int(zs[i]))
        assert abs(p[i] - op) <= 1e-7, (i, p[i], op)
        assert np.max(np.abs(res[i] - ob)) <= PT.TOL
        assert np.max(np.abs(res[i] - ob)) <= 1e-5 * max(1e-3, float(np.max(ob)))
        assert np.all(res[i][gm.occupancy == 1] == 0.0)
    g.close()


@pytest.mark.parametrize("cluster", ["1", "0"])
def test_belief_update_batch_C3_paths_and_alignment(Q, cluster, monkeypatch):
    """Batched Eq. 3 on a map with 16-byte rows (C3, 128x128): the one-pass cluster kernel
    (default) and the two-pass path against the oracle; then misaligned views (base pointer
    offset by one float, row stride not a multiple of 4) must take the unvectorised path and give
    the same results (no misaligned float4 access)."""
    monkeypatch.setenv("QVTS_BU_CLUSTER", cluster)
    gm = W.CONFIGS["C3"]["map"]()
    g = Q.Model(gm, action_mask=W.A8)
    o = O.Model.grid(gm, action_mask=W.A8)
    rng = np.random.default_rng(5)
    nb = 9
    B = np.stack([W.random_belief(gm, 200 + i, sparsity=0.5 if i % 3 == 0 else 0.0) for i in range(nb)]).astype(np.float32)
    acts = rng.choice(g.action_ids, size=nb)
    zs = np.zeros(nb, np.int32)
    for i in range(nb):
        P = o.marginal(o.predict(B[i].astype(np.float64), g.action_ids.index(acts[i])))
        zs[i] = int(np.argsort(P)[-1 - (i % 4)])
    out = torch.empty((nb, gm.occupancy.size), dtype=torch.float32, device="cuda")
    p = g.belief_update_batch(dev(B), acts, zs, out)
    res = out.cpu().numpy()
    for i in range(nb):
        ob, op = o.belief_update(B[i].astype(np.float64), g.action_ids.index(acts[i]), int(zs[i]))
        assert abs(p[i] - op) <= 1e-7
        assert np.max(np.abs(res[i] - ob)) <= PT.TOL
        assert np.all(res[i][gm.occupancy == 1] == 0.0)
    HW = gm.occupancy.size
    Bm = torch.zeros((nb, HW + 1), dtype=torch.float32, device="cuda")
    Bm[:, 1:] = dev(B)
    outm = torch.zeros((nb, HW + 1), dtype=torch.float32, device="cuda")
    pm = g.belief_update_batch(Bm[:, 1:], acts, zs, outm[:, 1:])
    # the misaligned views take the two-pass path (fp64 per-cell sums); the cluster path sums
    # fp32 per-thread partials of <= 48 cells: the normalisers agree to ~1e-9, both within 1e-7 of
    # the oracle above
    assert np.max(np.abs(np.asarray(pm) - np.asarray(p))) <= 1e-8
    assert np.max(np.abs(outm[:, 1:].cpu().numpy() - res)) <= 1e-7
    single = torch.empty(HW + 1, dtype=torch.float32, device="cuda")
    ps = g.belief_update(Bm[0, 1:], int(acts[0]), int(zs[0]), single[1:])
    assert abs(ps - p[0]) <= 1e-8 and np.max(np.abs(single[1:].cpu().numpy() - res[0])) <= 1e-7
    g.close()


@pytest.mark.parametrize("name,depth,n", [("C1", 2, 4), ("ragged", 3, 8), ("paper", 3, 16), ("C3", 3, 8),
                                          ("ragged", 1, 300), ("C1", 4, 2)])
def test_graph_plan_step_is_bit_identical(Q, name, depth, n, monkeypatch):
    """Small single-GPU plan steps run as one captured CUDA graph with device-side level counts:
    the same root Q bits, level counts and action as the level-synchronous path, across repeated
    (cached-graph) calls with different step keys; and the root Q matches the oracle."""
    gm = W.CONFIGS["C3"]["map"]() if name == "C3" else MAPS[name][0]()
    mask = W.A8 if name == "C3" else MAPS[name][1]
    g, o, Qo, _, _ = pair(Q, gm, mask)
    b32 = np.asarray(W.random_belief(gm, 11), np.float32)
    for step in (0, 1, 2):
        out = {}
        for flag in ("1", "0"):
            monkeypatch.setenv("QVTS_PLAN_GRAPH", flag)
            r = g.plan_step(dev(b32), depth, n, seed=9, step=step)
            out[flag] = (np.array(r.q_root[:g.n_actions]), list(r.n_vnodes[:depth + 1]), r.action)
        assert np.array_equal(out["1"][0], out["0"][0]) and out["1"][1] == out["0"][1] and out["1"][2] == out["0"][2]
    # the traced (level-synchronous) step of the same key against the oracle at 1e-5 with flagged-
    # draw replay; the graph step's root Q is bit-identical to it
    monkeypatch.setenv("QVTS_PLAN_GRAPH", "0")
    res, _, _ = run_parity(Q, gm, mask, depth, n, b32, seed=9, step=2, beliefs=(name != "C3"))
    assert list(res.q_root[:g.n_actions]) == list(out["1"][0])


@pytest.mark.parametrize("name,depth,n", [("C1", 2, 4), ("ragged", 3, 8), ("paper", 3, 16), ("C3", 3, 8),
                                          ("ragged", 1, 300)])
def test_leaf_mma_matches_scalar_leaf_and_oracle(Q, name, depth, n, monkeypatch):
    """The tensor-core leaf kernel (fp16 hi/lo split products, leafmma.cu) against the scalar fp32
    leaf kernel and the oracle: identical tree (counts, draws come from the non-leaf levels),
    every sampled leaf value and root Q within the north-star 1e-5."""
    gm = W.CONFIGS["C3"]["map"]() if name == "C3" else MAPS[name][0]()
    mask = W.A8 if name == "C3" else MAPS[name][1]
    g, o, Qo, _, _ = pair(Q, gm, mask)
    b32 = np.asarray(W.random_belief(gm, 13), np.float32)
    out = {}
    for flag in ("1", "0"):
        monkeypatch.setenv("QVTS_LEAF_MMA", flag)
        r = g.plan_step(dev(b32), depth, n, seed=4, step=1, want_trace=True)
        t = g.trace(with_draws=True, n_samples=n)
        lq = t["levels"][depth - 1]["q"]
        lv = np.array(t["leafV"]).reshape(-1, 16)
        sampled = np.array(lq["cnt"]) > 0
        out[flag] = (np.array(r.q_root[:g.n_actions]), list(r.n_vnodes[:depth + 1]), r.action,
                     np.where(sampled, lv, 0.0), np.array(lq["Q"]))
    assert out["1"][1] == out["0"][1]
    assert np.max(np.abs(out["1"][3] - out["0"][3])) <= PT.TOL      # every sampled leaf value
    assert np.max(np.abs(out["1"][4] - out["0"][4])) <= PT.TOL      # every leaf-level Q-node
    assert np.max(np.abs(out["1"][0] - out["0"][0])) <= PT.TOL
    # the tensor-core leaf tree against the oracle element by element (1e-5, flagged-draw replay)
    monkeypatch.setenv("QVTS_LEAF_MMA", "1")
    run_parity(Q, gm, mask, depth, n, b32, seed=4, step=1, beliefs=False)


@pytest.mark.parametrize("env", [{"QVTS_LEAF_KERNEL": "0"}, {"QVTS_LEAF_NSPLIT": "2"}, {"QVTS_LEAF_TMA": "0"},
                                 {"QVTS_CORRECT_STAGE": "0"}, {"QVTS_BAND_ROWS": "8"}],
                         ids=["hist_leaf", "leaf_split", "leaf_cp_async", "correct_unstaged", "band_rows_8"])
def test_alternative_kernel_paths_match_oracle(Q, env, monkeypatch):
    """Every run-time kernel option the library keeps (read per call; model-level for the band
    height) is a different code path to the same numbers: the k_hist<leaf> leaf level instead of
    k_leaf, k_leaf with its bands split over CTAs (band records summed by k_reduce), k_leaf's
    4-byte cp.async staging instead of TMA, k_correct without row staging, and 8-row hist bands.
    On a 160 x 96 map (two k_leaf bands, several hist bands, 16-byte rows) each runs the whole
    depth-3 tree against the oracle element by element with flagged-draw replay (c.5)."""
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    gm = W.random_map(160, 96, 0.2, seed=21)
    run_parity(Q, gm, W.A8, 3, 8, W.random_belief(gm, 13), seed=5, step=1)


def test_belief_update_batch_two_pass_tile_size(Q, monkeypatch):
    """The two-pass batched update with 256-group tiles (QVTS_BU_GROUPS, read per call; default
    2048) gives the cluster kernel's results on the C3 map: P to 1e-8, b' to 1e-7 (different
    fp32 prediction forms, Eq. 3)."""
    gm = W.CONFIGS["C3"]["map"]()
    g = Q.Model(gm, action_mask=W.A8)
    nb = 9
    B = np.stack([W.random_belief(gm, 700 + i) for i in range(nb)]).astype(np.float32)
    acts = np.array([g.action_ids[i % g.n_actions] for i in range(nb)], np.int32)
    zs = np.array([(3 * i) % 16 for i in range(nb)], np.int32)
    out1 = torch.empty((nb, gm.occupancy.size), dtype=torch.float32, device="cuda")
    out2 = torch.empty_like(out1)
    p1 = g.belief_update_batch(dev(B), acts, zs, out1)
    monkeypatch.setenv("QVTS_BU_CLUSTER", "0")
    monkeypatch.setenv("QVTS_BU_GROUPS", "256")
    p2 = g.belief_update_batch(dev(B), acts, zs, out2)
    assert np.max(np.abs(np.asarray(p1) - np.asarray(p2))) <= 1e-8
    assert float((out1 - out2).abs().max()) <= 1e-7
    g.close()
