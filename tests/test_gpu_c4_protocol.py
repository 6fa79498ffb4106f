"""SURVEY §8(c) c.5 at C4, the benchmarked configuration (BASELINE config 4: 256x256 Bernoulli(0.2)
map, A8, depth 4, n = 16, uniform root), launched as bench.py times it, against the fp64 oracle:

* every Q-node of levels 0-2 (8 + 472 + ~23K): R(b,a), P(z|b,a) (Eq. 3
  normaliser) and all n draws (Alg. 3-4): a draw may differ only
  where the oracle flags it (CDF gap < 1e-6, reading R11); the oracle's beliefs follow the GPU's
  tree (Eq. 3 with the GPU's z on every edge, i.e. c.5 replay);
* a seeded 1% of the level-3 V-nodes: their 8 leaf Q-nodes' R, P and draws, V (Alg. 7) and Q
  (Alg. 6 with gamma) from the oracle's own subtree recursion with the GPU's draws replayed where
  the oracle flags them; and for a subset every sampled leaf's Q_MDP value (Eq. 4);
* 16 full level-2 subtrees (V of the level-2 node from the oracle's depth-2 recursion);
* 16 beliefs per level, element by element (Eq. 3);
* the flagged-draw count exported by the library (qvts_plan_result.n_flag_candidates), and the
  backup identity Q = R + gamma sum (f/n) V on the GPU's own arrays.

Tolerances are the north star's: values 1e-5 absolute, non-flagged draws bit-exact.  The oracle
work is spread over the host's cores with forked workers (each walks its own level-1 subtrees)."""
import multiprocessing as mp
import os

import numpy as np
import pytest

import oracle as O
import workloads as W
from tests import parity as PT

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

_G = {}   # read by the forked workers


@pytest.fixture(scope="module")
def Q():
    assert torch.cuda.is_available(), "GPU tests need CUDA"
    from paper_1810_00204_b200 import qvts
    qvts.lib()
    return qvts


def _qnode_check(o, b, ai, qpath, n, gq_R, gq_P, gq_z, seed=1):
    """R, P and draws of one Q-node against the oracle on belief b."""
    P, R, z, flag, cnt = o.qnode_sample(b, ai, qpath, n, seed=seed)
    mism = gq_z != z
    return dict(eR=abs(gq_R - R), eP=float(np.max(np.abs(gq_P - P))), nonflag=int(np.sum(mism & ~flag)),
                flagmis=int(np.sum(mism & flag)), flags=int(np.sum(flag)), draws=len(z))


def _merge(acc, r):
    for k, v in r.items():
        if k.startswith("e"):
            acc[k] = max(acc.get(k, 0.0), v)
        else:
            acc[k] = acc.get(k, 0) + v


def _replay_of(qlev, level, qs, n):
    """The GPU's draws of Q-nodes qs at `level` as replay entries (the oracle takes one only where
    it flags that draw itself and the category borders the near boundary, c.5 step 3)."""
    ent = []
    for q in qs:
        p = int(qlev[level]["path"][q])
        for j in range(n):
            ent.append((p, j, int(qlev[level]["z"][q][j])))
    return ent


def _children(vlev, level, q):
    """Indices of the level-`level` V-nodes whose parent Q-node (at level-1) is q."""
    return _G["kids"][level].get(q, [])


def _worker(unit):
    g = _G
    o, Qo, na, n, qlev, vlev, leafV = g["o"], g["Qo"], g["na"], g["n"], g["qlev"], g["vlev"], g["leafV"]
    i1, s3, s2full, bel_check = unit
    acc = {}
    beliefs_out = {}
    b0 = g["b0"]
    q0 = int(vlev[1]["parent_q"][i1])
    b1, _ = o.belief_update(b0, q0 % na, int(vlev[1]["z"][i1]))
    bel = {(1, i1): b1}
    # level-1 Q-nodes and their level-2 children (all of them: scalars of levels <= 2)
    for aj in range(na):
        q1 = i1 * na + aj
        _merge(acc, _qnode_check(o, b1, aj, int(qlev[1]["path"][q1]), n, qlev[1]["R"][q1], qlev[1]["P"][q1],
                                 qlev[1]["z"][q1]))
        for i2 in _children(vlev, 2, q1):
            b2, _ = o.belief_update(b1, aj, int(vlev[2]["z"][i2]))
            bel[(2, i2)] = b2
            for aj2 in range(na):
                q2 = i2 * na + aj2
                _merge(acc, _qnode_check(o, b2, aj2, int(qlev[2]["path"][q2]), n, qlev[2]["R"][q2], qlev[2]["P"][q2],
                                         qlev[2]["z"][q2]))
    # full level-2 subtrees: V of the level-2 node by the oracle's depth-2 recursion
    for i2 in s2full:
        qs2 = list(range(i2 * na, (i2 + 1) * na))
        rep = _replay_of(qlev, 2, qs2, n)
        for q2 in qs2:
            rep += _replay_of(qlev, 3, [i3 * na + a3 for i3 in _children(vlev, 3, q2) for a3 in range(na)], n)
        Vo, qv = o.vnode_value(Qo, bel[(2, i2)], int(vlev[2]["path"][i2]), 2, 4, n, seed=1, replay=rep)
        acc["eV2"] = max(acc.get("eV2", 0.0), abs(vlev[2]["V"][i2] - Vo))
        acc["eQ2"] = max(acc.get("eQ2", 0.0), float(np.max(np.abs(qlev[2]["Q"][qs2[0]:qs2[-1] + 1] - qv))))
        acc["n_sub2"] = acc.get("n_sub2", 0) + 1
    # the sampled level-3 V-nodes
    for k, i3 in enumerate(s3):
        q2 = int(vlev[3]["parent_q"][i3])
        i2 = q2 // na
        b3, _ = o.belief_update(bel[(2, i2)], q2 % na, int(vlev[3]["z"][i3]))
        bel[(3, i3)] = b3
        qs3 = list(range(i3 * na, (i3 + 1) * na))
        for q3 in qs3:
            _merge(acc, _qnode_check(o, b3, q3 % na, int(qlev[3]["path"][q3]), n, qlev[3]["R"][q3], qlev[3]["P"][q3],
                                     qlev[3]["z"][q3]))
        Vo, qv = o.vnode_value(Qo, b3, int(vlev[3]["path"][i3]), 3, 4, n, seed=1, replay=_replay_of(qlev, 3, qs3, n))
        acc["eV3"] = max(acc.get("eV3", 0.0), abs(vlev[3]["V"][i3] - Vo))
        acc["eQ3"] = max(acc.get("eQ3", 0.0), float(np.max(np.abs(qlev[3]["Q"][qs3[0]:qs3[-1] + 1] - qv))))
        acc["n_sub3"] = acc.get("n_sub3", 0) + 1
        if k < 2:          # every sampled leaf of this node: Q_MDP value of the child belief (Eq. 4)
            for q3 in qs3:
                for z in np.flatnonzero(qlev[3]["cnt"][q3]):
                    b4, _ = o.belief_update(b3, q3 % na, int(z))
                    v, _ = o.qmdp_value(Qo, b4)
                    acc["eleaf"] = max(acc.get("eleaf", 0.0), abs(leafV[q3][z] - v))
                    acc["n_leaf"] = acc.get("n_leaf", 0) + 1
    for key in bel_check:
        if key in bel:
            beliefs_out[key] = bel[key]
    return acc, beliefs_out


def test_C4_comparison_protocol(Q):
    cfg = W.CONFIGS["C4"]
    gm = cfg["map"]()
    D, n = cfg["depth"], cfg["n"]
    g = Q.Model(gm, action_mask=W.A8)
    code, _, _ = g.value_iteration(1e-9)
    assert code == 0
    o = O.Model.grid(gm, action_mask=W.A8)
    st, _, Qo, _, _ = o.value_iteration(1e-9)
    assert st == O.OK
    b32 = W.uniform_belief(gm, np.float32)
    res = g.plan_step(torch.tensor(b32, device="cuda"), D, n, seed=1, want_trace=True)
    na = g.n_actions
    _, nv, nqw = Q.qvts_trace_counts(g.h)
    vlev = [Q.qvts_trace_vnodes(g.h, d, nv[d]) for d in range(D)]
    qlev = [Q.qvts_trace_qnodes(g.h, d, nqw[d] * na, n, True) for d in range(D)]
    leafV = Q.qvts_trace_leaf_values(g.h, nqw[D - 1] * na)
    assert nqw[3] == nv[3] and nv[3] > 100_000
    rng = np.random.default_rng(2024)
    kids = {d: {} for d in (2, 3)}
    for d in (2, 3):
        for i, q in enumerate(vlev[d]["parent_q"]):
            kids[d].setdefault(int(q), []).append(i)
    # level-1 ancestor of every level-2 / level-3 V-node
    anc2 = (vlev[2]["parent_q"] // na).astype(np.int64)
    anc3 = anc2[(vlev[3]["parent_q"] // na).astype(np.int64)]
    s3 = np.sort(rng.choice(nv[3], size=max(1, nv[3] // 100), replace=False))        # 1% of level 3
    s2 = np.sort(rng.choice(nv[2], size=16, replace=False))
    bchk = {1: rng.choice(nv[1], size=16, replace=False), 2: rng.choice(nv[2], size=16, replace=False),
            3: rng.choice(s3, size=16, replace=False)}
    units = []
    for i1 in range(nv[1]):
        units.append((i1, [int(i) for i in s3 if anc3[i] == i1], [int(i) for i in s2 if anc2[i] == i1],
                      [(d, int(i)) for d in (1, 2, 3) for i in bchk[d]
                       if (d == 1 and i == i1) or (d == 2 and anc2[i] == i1) or (d == 3 and anc3[i] == i1)]))
    gpu_bel = {(d, int(i)): Q.qvts_trace_belief(g.h, d, int(i), g.n_cells).astype(np.float64)
               for d in (1, 2, 3) for i in bchk[d]}
    _G.update(o=o, Qo=Qo, na=na, n=n, qlev=qlev, vlev=vlev, leafV=leafV, b0=b32.astype(np.float64), kids=kids)
    acc = {}
    # level 0 in this process
    for aj in range(na):
        _merge(acc, _qnode_check(o, b32.astype(np.float64), aj, int(qlev[0]["path"][aj]), n, qlev[0]["R"][aj],
                                 qlev[0]["P"][aj], qlev[0]["z"][aj]))
    ncpu = max(1, min(len(units), os.cpu_count() or 1))
    with mp.get_context("fork").Pool(ncpu) as pool:
        outs = pool.map(_worker, sorted(units, key=lambda u: -len(u[1])), chunksize=1)
    obel = {}
    for a, bo in outs:
        _merge(acc, a)
        obel.update(bo)
    ebel = max(float(np.max(np.abs(gpu_bel[k] - obel[k]))) for k in gpu_bel)
    print(f"\nC4 c.5 protocol: {acc.get('draws', 0)} draws compared, {acc.get('flags', 0)} flagged by the "
          f"oracle, {acc.get('flagmis', 0)} flagged mismatches (replayed), GPU flag candidates "
          f"{res.n_flag_candidates}; max |dR| {acc['eR']:.2e} |dP| {acc['eP']:.2e} |dV3| {acc['eV3']:.2e} "
          f"|dQ3| {acc['eQ3']:.2e} |dV2| {acc['eV2']:.2e} |dQ2| {acc['eQ2']:.2e} |dleaf| {acc['eleaf']:.2e} "
          f"({acc['n_leaf']} leaves) |dbelief| {ebel:.2e}; {acc['n_sub3']} level-3 and {acc['n_sub2']} level-2 subtrees")
    assert acc["nonflag"] == 0, f"{acc['nonflag']} non-flagged draw mismatches"
    assert acc["n_sub3"] == len(s3) and acc["n_sub2"] == 16 and len(obel) == len(gpu_bel)
    for k in ("eR", "eV3", "eQ3", "eV2", "eQ2", "eleaf"):
        assert acc[k] <= PT.TOL, (k, acc[k])
    assert acc["eP"] <= 1e-6
    assert ebel <= PT.TOL
    assert res.n_flag_candidates > 0
    # backup identity at every level from the GPU's own arrays (fp64 recompute), and the root
    for d in range(D - 2, -1, -1):
        lq, lc = qlev[d], vlev[d + 1]
        off = np.concatenate([[0], np.cumsum([int((c > 0).sum()) for c in lq["cnt"]])])
        for qi in rng.integers(0, len(lq["R"]), size=min(500, len(lq["R"]))):
            s = sum((lc["f"][c] / n) * lc["V"][c] for c in range(off[qi], off[qi + 1]))
            assert abs(lq["R"][qi] + 0.95 * s - lq["Q"][qi]) <= 1e-9
    assert np.max(np.abs(np.array(res.q_root[:na]) - qlev[0]["Q"])) == 0.0
    g.close()
