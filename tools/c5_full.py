"""C5 as SURVEY §8(d) d.1 defines it: random(256,256,0.2,seed=5), A9, 1024 episodes, D=3, n=8,
max_steps 1000, uniform b0 -- one batched qvts_run_episodes call on one B200.  Prints one JSON
object: wall time, episodes/s, episode-steps/s, outcome counts, success rate."""
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

E = int(os.environ.get("EPISODES", "1024"))
MS = int(os.environ.get("MAX_STEPS", "1000"))
MAP_SEED = int(os.environ.get("MAP_SEED", "5"))          # SURVEY d.1: C5 x 3 map seeds as separate runs
gm = W.random_map(256, 256, 0.2, seed=MAP_SEED)
m = Q.Model(gm, action_mask=W.A9)
m.value_iteration(1e-9)
m.run_episodes(8, max_steps=5, planner=Q.QVTS_PLANNER_QVTS, depth=3, n_samples=8, seed=99)   # warm
torch.cuda.synchronize()
t0 = time.perf_counter()
rec, _ = m.run_episodes(E, max_steps=MS, stop_patience=3, planner=Q.QVTS_PLANNER_QVTS, depth=3, n_samples=8, seed=1)
torch.cuda.synchronize()
dt = time.perf_counter() - t0
steps = int(rec["steps"].sum())
oc = {str(k): int((rec["outcome"] == k).sum()) for k in range(4)}
print(json.dumps({"config": f"C5: random(256,256,0.2,seed={MAP_SEED}), A9, D=3, n=8, {E} episodes, max_steps {MS}, stop_patience 3, uniform b0",
                  "episodes": E, "wall_s": dt, "episodes_per_s": E / dt, "episode_steps": steps,
                  "episode_steps_per_s": steps / dt, "mean_steps": steps / E, "outcomes": oc,
                  "success_rate": oc["0"] / E, "mean_collisions": float(rec["collisions"].mean()),
                  "mean_return": float(rec["disc_return"].mean())}), flush=True)
