"""Config 2 with the paper's own planner: the anytime best-first QVTS (Alg. 1 with the inner
best-first loop, FIB upper / PBVI lower leaves, AEMS rule, tree reuse by s.update(a, z)) in a
closed loop on the paper-style 50x50 maps, beside the MDP and A* baselines of
tools/config2_episodes.py.  The environment (true motion with collisions, sensor noise, the
stop rule of readings R26/R27) is simulated here on the host with numpy's seeded generator --
an application driver on top of the public API, not part of the GPU path.  Prints JSON lines."""
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import workloads as W  # noqa: E402
from paper_1810_00204_b200 import qvts as Q  # noqa: E402

E = int(os.environ.get("EPISODES", "60"))
BUDGET = int(os.environ.get("BF_EXPANSIONS", "64"))
MAX_STEPS, PATIENCE, GAMMA = 500, 3, 0.95
P_INT, P_STAY, P_LAT, ACC = 0.8, 0.1, 0.05, 0.95
RING = [0, 1, 2, 5, 8, 7, 6, 3]


def step_env(rng, gm, x, a):
    """True motion ~ T'(x,a,.) (pre-clamp): a blocked target is a collision and x stays."""
    H, Wd = gm.height, gm.width
    if a == 4:
        k = 4
    else:
        i = RING.index(a)
        ks = [a, 4, RING[(i + 1) % 8], RING[(i - 1) % 8]]
        k = ks[rng.choice(4, p=[P_INT, P_STAY, P_LAT, P_LAT])]
    if k == 4:
        return x, False
    r, c = divmod(x, Wd)
    rr, cc = r + k // 3 - 1, c + k % 3 - 1
    if rr < 0 or rr >= H or cc < 0 or cc >= Wd or gm.occupancy[rr * Wd + cc]:
        return x, True
    return rr * Wd + cc, False


def observe(rng, sig, x):
    flips = rng.random(4) >= ACC
    return int(sig[x]) ^ int(sum(1 << b for b in range(4) if flips[b]))


def episode(m, gm, R, sig, b0, rng, seed, ep):
    free = np.flatnonzero(gm.occupancy == 0)
    x = int(rng.choice(free, p=b0[free] / b0[free].sum()))
    b = torch.tensor(b0.astype(np.float32), device="cuda")
    nb = torch.empty_like(b)
    ret, disc, streak, coll, reuse = 0.0, 1.0, 0, 0, False
    for t in range(MAX_STEPS):
        res = m.plan_best_first(None if reuse else b, 16, BUDGET, max_depth=8, seed=seed, step=t, episode=ep,
                                reuse=reuse)
        a = res.action
        j = m.action_ids.index(a)
        ret += disc * float(R[j, x])
        disc *= GAMMA
        if a == 4:
            streak += 1
            if streak >= PATIENCE:
                return (0 if x == gm.goal else 1), t + 1, coll, ret
        else:
            streak = 0
        x, hit = step_env(rng, gm, x, a)
        coll += int(hit)
        z = observe(rng, sig, x)
        try:
            m.belief_update(b, a, z, nb)
        except Q.QvtsError:
            return 3, t + 1, coll, ret
        b, nb = nb, b
        reuse = m.bf_advance(a, z)
    return 2, MAX_STEPS, coll, ret


out = {"config": f"C2 maps paper_style(50,50,6,12,seed), A9, best-first QVTS: n=16, {BUDGET} expansions per step, "
                 "max_depth 8, tree reuse; PBVI 4 rounds / 32 points / 30 sweeps from uniform b0; max_steps 500, "
                 "patience 3", "episodes_per_map": E, "maps": {}}
for mseed in (1, 2, 3):
    gm = W.paper_style(50, 50, 6, 12, seed=mseed)
    m = Q.Model(gm, action_mask=W.A9)
    m.value_iteration()
    m.fib_iteration()
    b0 = W.uniform_belief(gm)
    Q.qvts_pbvi(m.h, torch.tensor(b0.astype(np.float32), device="cuda"), 4, 32, 1, 30)
    R, sig = m.tables()
    R = np.asarray(R, np.float64).reshape(m.n_actions, -1)
    rng = np.random.default_rng(1000 + mseed)
    recs = []
    t0 = time.perf_counter()
    for ep in range(E):
        recs.append(episode(m, gm, R, sig, b0, rng, mseed, ep))
    dt = time.perf_counter() - t0
    oc = np.array([r[0] for r in recs])
    steps = np.array([r[1] for r in recs])
    ok = oc == 0
    res = {"failure_rate": float(1 - ok.mean()), "steps_mean": float(steps.mean()),
           "steps_success_mean": float(steps[ok].mean()) if ok.any() else None,
           "collisions_mean": float(np.mean([r[2] for r in recs])),
           "disc_return_mean": float(np.mean([r[3] for r in recs])),
           "outcomes": {str(k): int((oc == k).sum()) for k in range(4)},
           "wall_s": dt, "ms_per_episode_step": 1e3 * dt / max(1, steps.sum())}
    out["maps"][mseed] = {"QVTS-best-first": res}
    print(json.dumps({"map_seed": mseed, "QVTS-best-first": res}), flush=True)
    m.close()
agg = {k: float(np.mean([out["maps"][s]["QVTS-best-first"][k] for s in out["maps"]]))
       for k in ("failure_rate", "steps_mean", "collisions_mean", "disc_return_mean")}
out["mean_over_maps"] = agg
print(json.dumps({"mean_over_maps": agg}), flush=True)
json.dump(out, open(os.path.join(ROOT, "gpurun_out", "config2_bestfirst.json"), "w"), indent=1)
