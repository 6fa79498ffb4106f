"""Why does QVTS fail on config-2 map 1 (paper_style(50,50,6,12,seed=1))?  VERDICT r01 item 7,
against SURVEY pin P16 (Table I ordering).  Runs the closed loop (Alg. 1,
qvts_run_episodes) with logs and separates the candidate causes:

* the stop rule (reading R26: `stop_patience` consecutive stays, success iff the true state is the
  goal): patience 1 / 2 / 3;
* the Q_MDP leaf (reading R14) through the look-ahead depth: D = 2, 3, 4;
* the map (global localisation): point-mass starts (the robot knows where it starts) for QVTS and
  for the MDP baseline;

and reports for every variant the outcome counts, the failure rate with and without wrong stops
counted as failures, the rate of episodes whose true state ever reached the goal, and for the
step-capped episodes how the last 100 steps were spent (at the goal, staying, within 2 cells), plus
the belief at the cap (Eq. 3 replayed over the logged (a, z) with the oracle: mass on the goal,
max mass, entropy).  Writes gpurun_out/config2_diagnosis.json."""
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle as O  # noqa: E402  (test/measurement infrastructure: replays beliefs from the logs)
import workloads as W  # noqa: E402
from paper_1810_00204_b200 import qvts as Q  # noqa: E402

E = int(os.environ.get("EPISODES", "60"))
MS = 500
gm = W.paper_style(50, 50, 6, 12, seed=1)
H, Wd = gm.height, gm.width
m = Q.Model(gm, action_mask=W.A9)
m.value_iteration()
om = O.Model.grid(gm, action_mask=W.A9)
goal = gm.goal
gr, gc = divmod(goal, Wd)


def cheb(x):
    r, c = divmod(int(x), Wd)
    return max(abs(r - gr), abs(c - gc))


def run(name, planner, depth=3, n=16, patience=3, b0=None, episodes=E, seed=1, replay_beliefs=True):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    b0_dev = torch.tensor(np.asarray(b0, np.float32), device="cuda") if b0 is not None else None
    rec, logs = m.run_episodes(episodes, max_steps=MS, stop_patience=patience, planner=planner, depth=depth,
                               n_samples=n, seed=seed, b0_dev=b0_dev, logs=True)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    oc = rec["outcome"]
    st = logs["states"]
    reached = np.array([np.any(st[e][: rec["steps"][e]] == goal) for e in range(episodes)])
    out = {"planner": ["QVTS", "MDP", "A*"][planner], "depth": depth, "n": n, "patience": patience,
           "start": "uniform" if b0 is None else "point mass", "episodes": episodes,
           "outcomes": {"success": int((oc == 0).sum()), "wrong_stop": int((oc == 1).sum()),
                        "step_cap": int((oc == 2).sum())},
           "failure_rate_incl_wrong_stop": float((oc != 0).mean()),
           "failure_rate_excl_wrong_stop": float((oc == 2).mean()),
           "reached_goal_rate": float(reached.mean()),
           "steps_mean": float(rec["steps"].mean()), "wall_s": dt}
    capped = np.flatnonzero(oc == 2)
    if len(capped):
        at_goal, stays, near = [], [], []
        for e in capped:
            s = st[e][MS - 100: MS]
            a = logs["actions"][e][MS - 100: MS]
            at_goal.append(float(np.mean(s == goal)))
            stays.append(float(np.mean(a == 4)))
            near.append(float(np.mean([cheb(x) <= 2 for x in s])))
        out["capped_last100"] = {"frac_at_goal": float(np.mean(at_goal)), "frac_stay_actions": float(np.mean(stays)),
                                 "frac_within_2_of_goal": float(np.mean(near))}
        if replay_beliefs:
            bstats = []
            for e in capped[:12]:
                b = W.uniform_belief(gm) if b0 is None else np.asarray(b0, np.float64)
                for k in range(MS):
                    a = int(logs["actions"][e][k])
                    z = int(logs["obs"][e][k])
                    b, _ = om.belief_update(b, om.action_ids.index(a), z)
                nz = b[b > 0]
                bstats.append({"mass_on_goal": float(b[goal]), "max_mass": float(b.max()),
                               "argmax_cheb_to_goal": cheb(int(np.argmax(b))),
                               "true_cheb_to_goal": cheb(int(st[e][MS - 1])),
                               "entropy_nats": float(-(nz * np.log(nz)).sum())})
            out["capped_final_belief"] = {k: float(np.mean([s[k] for s in bstats])) for k in bstats[0]}
    print(json.dumps({name: out}), flush=True)
    return out


res = {"map": "paper_style(50,50,6 walls,12 pillars,seed=1), A9, goal cell %d (row %d, col %d)" % (goal, gr, gc),
       "max_steps": MS}
res["qvts_D3_p3"] = run("qvts_D3_p3", 0)
res["qvts_D3_p1"] = run("qvts_D3_p1", 0, patience=1)
res["qvts_D3_p2"] = run("qvts_D3_p2", 0, patience=2)
res["qvts_D2_p3"] = run("qvts_D2_p3", 0, depth=2)
res["qvts_D4_p3"] = run("qvts_D4_p3", 0, depth=4, n=8, episodes=min(E, 20))
res["mdp_p3"] = run("mdp_p3", 1, replay_beliefs=False)
res["astar_p3"] = run("astar_p3", 2, replay_beliefs=False)
# point-mass starts: 6 start cells x E/6 episodes, QVTS and MDP
pm = {"QVTS": [], "MDP": []}
for k in range(6):
    b0 = W.point_belief(gm, W.free_cell(gm, 100 + k))
    pm["QVTS"].append(run(f"qvts_point_{k}", 0, b0=b0, episodes=max(1, E // 6), seed=10 + k, replay_beliefs=False))
    pm["MDP"].append(run(f"mdp_point_{k}", 1, b0=b0, episodes=max(1, E // 6), seed=10 + k, replay_beliefs=False))
for name, lst in pm.items():
    tot = sum(r["episodes"] for r in lst)
    res[f"{name.lower()}_point_starts"] = {
        "episodes": tot,
        "success": sum(r["outcomes"]["success"] for r in lst),
        "wrong_stop": sum(r["outcomes"]["wrong_stop"] for r in lst),
        "step_cap": sum(r["outcomes"]["step_cap"] for r in lst),
        "steps_mean": float(np.mean([r["steps_mean"] for r in lst])),
        "per_start": lst}
os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
json.dump(res, open(os.path.join(ROOT, "gpurun_out", "config2_diagnosis.json"), "w"), indent=1)
