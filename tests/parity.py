"""GPU-vs-oracle comparison helpers.  Test infrastructure only."""
from __future__ import annotations

import numpy as np

import oracle as O

TOL = 1e-5          # beliefs, P, R, Q, V: absolute (north star)
TIE = 1e-6          # chosen actions may differ only across a tie within this (north star)


def gpu_tree(model, n, with_beliefs=False, with_states=False):
    """Flatten the GPU trace into dicts keyed by tree path (with_states: the ancestral sampler's
    state index x of every draw, for the c.5 replay of flagged state draws)."""
    t = model.trace(with_draws=True, n_samples=n, beliefs=with_beliefs, with_states=with_states)
    D = t["depth"]
    na = model.n_actions
    q, v, bel = {}, {}, {}
    for d in range(D):
        lq, lv = t["levels"][d]["q"], t["levels"][d]["v"]
        for i in range(len(lq["path"])):
            q[int(lq["path"][i])] = dict(level=d, idx=i, R=lq["R"][i], P=lq["P"][i], cnt=lq["cnt"][i],
                                         Q=lq["Q"][i], z=lq["z"][i],
                                         x=lq["x"][i] if with_states else None)
        if d > 0:
            for i in range(len(lv["path"])):
                v[int(lv["path"][i])] = dict(level=d, V=lv["V"][i], z=int(lv["z"][i]), f=int(lv["f"][i]))
                if with_beliefs:
                    bel[int(lv["path"][i])] = t["levels"][d]["v"]["belief"][i]
    # leaf V-nodes (level D) from the leaf values of the last Q-level
    lq = t["levels"][D - 1]["q"]
    for i in range(len(lq["path"])):
        for z in range(16):
            if lq["cnt"][i][z]:
                v[O.vpath_child(int(lq["path"][i]), D - 1, z)] = dict(level=D, V=t["leafV"][i][z], z=z,
                                                                     f=int(lq["cnt"][i][z]))
    return q, v, bel, na


def oracle_tree(res):
    t = res.trace
    q = {}
    for i in range(len(t.q_path)):
        q[int(t.q_path[i])] = dict(level=int(t.q_level[i]), R=t.q_R[i], P=t.q_P[i], cnt=t.q_cnt[i], Q=t.q_Q[i],
                                   z=t.q_z[i], flag=t.q_flag[i])
    v = {int(t.v_path[i]): dict(level=int(t.v_level[i]), V=t.v_V[i], z=int(t.v_z[i]), f=int(t.v_f[i]))
         for i in range(len(t.v_path))}
    return q, v, t.v_belief


def draw_mismatches(gq, oq):
    """Mismatched draws per Q-node path; raises on a mismatch of a non-flagged draw.  Replay
    entries carry the GPU's z and, for the ancestral sampler, its state index x (the oracle then
    takes x only if it borders the flagged boundary and recomputes x' and z from it)."""
    replay, n_flag_mismatch = [], 0
    for p, o in oq.items():
        g = gq.get(p)
        if g is None:
            continue
        diff = np.flatnonzero(g["z"] != o["z"])
        for j in diff:
            if not o["flag"][j]:
                raise AssertionError(f"non-flagged draw mismatch at path {p:#x} sample {j}: "
                                     f"gpu {g['z'][j]} oracle {o['z'][j]}")
            if g.get("x") is not None:
                replay.append((p, int(j), int(g["z"][j]), int(g["x"][j])))
            else:
                replay.append((p, int(j), int(g["z"][j])))
            n_flag_mismatch += 1
    return replay, n_flag_mismatch


def compare_trees(gq, gv, oq, ov, gbel=None, obel=None, tol=TOL):
    """Element-wise comparison; returns a dict of max errors."""
    assert set(gq) == set(oq), f"Q-node sets differ: {len(set(gq) ^ set(oq))} paths"
    assert set(gv) == set(ov), f"V-node sets differ: {len(set(gv) ^ set(ov))} paths"
    err = dict(R=0.0, P=0.0, Q=0.0, V=0.0, belief=0.0)
    for p, o in oq.items():
        g = gq[p]
        assert np.array_equal(g["cnt"], o["cnt"]), f"counts differ at {p:#x}"
        err["R"] = max(err["R"], abs(g["R"] - o["R"]))
        err["P"] = max(err["P"], float(np.max(np.abs(g["P"] - o["P"]))))
        err["Q"] = max(err["Q"], abs(g["Q"] - o["Q"]))
    for p, o in ov.items():
        g = gv[p]
        assert g["f"] == o["f"] and g["z"] == o["z"]
        err["V"] = max(err["V"], abs(g["V"] - o["V"]))
    if gbel is not None and obel is not None:
        for p, b in obel.items():
            err["belief"] = max(err["belief"], float(np.max(np.abs(gbel[p].astype(np.float64) - b))))
    for k, e in err.items():
        assert e <= tol, f"{k} error {e:.3e} > {tol}"
    return err


def check_action(action_gpu, action_or, qroot_or, action_ids):
    if action_gpu == action_or:
        return
    ia, io = action_ids.index(action_gpu), action_ids.index(action_or)
    assert abs(qroot_or[ia] - qroot_or[io]) <= TIE, "chosen actions differ beyond a tie"
