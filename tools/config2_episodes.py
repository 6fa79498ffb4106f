"""BASELINE config 2: paper-style ~50x50 maps, 9 actions, depth 3, full episodes to the goal;
success (failure) rate, steps, collisions and discounted return of QVTS vs MDP vs A* (Table I
shape; ordering-level only, the paper's map is unpublished)."""
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
out = {"config": "C2: paper_style(50,50,6 walls,12 pillars), A9, depth 3, n=16, max_steps 500, patience 3",
       "episodes_per_planner_per_map": E, "maps": {}}
for seed in (1, 2, 3):
    gm = W.paper_style(50, 50, 6, 12, seed=seed)
    m = Q.Model(gm, action_mask=W.A9)
    m.value_iteration()
    res = {}
    for name, pl in (("A*", 2), ("MDP", 1), ("QVTS", 0)):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        rec, _ = m.run_episodes(E, max_steps=500, stop_patience=3, planner=pl, depth=3, n_samples=16, seed=seed)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        ok = rec["outcome"] == 0
        res[name] = {"failure_rate": float(1 - ok.mean()), "steps_mean": float(rec["steps"].mean()),
                     "steps_success_mean": float(rec["steps"][ok].mean()) if ok.any() else None,
                     "collisions_mean": float(rec["collisions"].mean()),
                     "disc_return_mean": float(rec["disc_return"].mean()),
                     "disc_return_std": float(rec["disc_return"].std()),
                     "outcomes": {str(k): int((rec["outcome"] == k).sum()) for k in range(4)},
                     "wall_s": dt, "ms_per_episode_step": 1e3 * dt / max(1, rec["steps"].sum()) * E}
    out["maps"][seed] = res
    print(json.dumps({"map_seed": seed, **res}), flush=True)
agg = {}
for name in ("A*", "MDP", "QVTS"):
    agg[name] = {k: float(np.mean([out["maps"][s][name][k] for s in out["maps"]]))
                 for k in ("failure_rate", "steps_mean", "collisions_mean", "disc_return_mean")}
out["mean_over_maps"] = agg
print(json.dumps({"mean_over_maps": agg}), flush=True)
json.dump(out, open(os.path.join(ROOT, "gpurun_out", "config2.json"), "w"), indent=1)
