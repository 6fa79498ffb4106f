"""Small-config exercise of every library entry point and kernel option, for compute-sanitizer
(memcheck / racecheck / synccheck / initcheck; SURVEY §4 layer 5).  Run as
    compute-sanitizer --tool <tool> python tools/sanitize_small.py [quick]
Covers: VI, FIB, PBVI, belief_update (single, batch), plan_step (Q_MDP and FIB leaves, marginal
and ancestral samplers, graph-captured and level-synchronous, the k_hist leaf path, k_leaf's
cp.async staging fallback and band split, the opt-in tensor-core leaf kernel, k_correct staged
and unstaged), belief_update_batch on both paths, best-first planning with tree reuse and the
three episode planners."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import workloads as W  # noqa: E402
from paper_1810_00204_b200 import qvts as Q  # noqa: E402

quick = len(sys.argv) > 1 and sys.argv[1] == "quick"
maps = [(W.CONFIGS["C1"]["map"](), W.A4), (W.random_map(13, 17, 0.2, seed=2), W.A8),
        (W.random_map(24, 32, 0.2, seed=3), W.A8), (W.paper_style(30, 30, 3, 5, seed=1), W.A9)]
for gm, mask in maps:
    m = Q.Model(gm, action_mask=mask)
    m.value_iteration(1e-9)
    m.fib_iteration(1e-9)
    b = torch.tensor(W.uniform_belief(gm, np.float32), device="cuda")
    out = torch.empty_like(b)
    m.belief_update(b, m.action_ids[0], 3, out)
    bb = torch.stack([b, out])
    ob = torch.empty_like(bb)
    m.belief_update_batch(bb, [m.action_ids[1], m.action_ids[0]], [2, 5], ob)
    os.environ["QVTS_BU_CLUSTER"] = "0"                     # the two-pass path too
    m.belief_update_batch(bb, [m.action_ids[1], m.action_ids[0]], [2, 5], ob)
    os.environ.pop("QVTS_BU_CLUSTER")
    for leaf in (0, 1):
        for sampler in ((0, 1) if not quick else (0,)):
            m.plan_step(b, 2, 8, seed=1, want_trace=True, leaf_bound=leaf, sampler=sampler)
            m.trace(with_draws=True, n_samples=8, beliefs=True)
    for env in ({}, {"QVTS_PLAN_GRAPH": "0"}, {"QVTS_LEAF_KERNEL": "0", "QVTS_PLAN_GRAPH": "0"},
                {"QVTS_LEAF_TMA": "0", "QVTS_PLAN_GRAPH": "0"}, {"QVTS_LEAF_NSPLIT": "4", "QVTS_PLAN_GRAPH": "0"},
                {"QVTS_LEAF_MMA": "1", "QVTS_PLAN_GRAPH": "0"}, {"QVTS_LEAF_MMA": "1"},
                {"QVTS_CORRECT_STAGE": "0", "QVTS_PLAN_GRAPH": "0"}):
        old = {k: os.environ.get(k) for k in env}
        os.environ.update(env)
        m.plan_step(b, 3, 4, seed=2, step=1)
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v
    m.pbvi(b, expansions=2, max_points=6, seed=1, sweeps=4)
    r = m.plan_best_first(b, 4, 12, max_depth=4, seed=1)
    m.trace_best_first()
    if r.n_expansions > 0:
        try:
            m.bf_advance(r.action, 0)
        except Exception:
            pass
        m.plan_best_first(None, 4, 6, max_depth=4, seed=1, reuse=True)
    for pl in ((0, 1, 2) if not quick else (0,)):
        m.run_episodes(3, max_steps=8, planner=pl, depth=2, n_samples=4, seed=1)
    m.close()
torch.cuda.synchronize()
print("sanitize_small ok")
