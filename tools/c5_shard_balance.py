"""Projected scaling of the C5 episode batch (1024 episodes sharded e = r mod G)
from one GPU: each rank's episodes run in turn (one batched qvts_run_episodes call per rank,
the record exchange replaced by a no-op callback) and are wall-timed; the projected G-GPU batch
time is the slowest rank plus one all-reduce of the record array, so speedup(G) = T(1) / max_r T_r.
Outcome counts summed over ranks equal the single-GPU batch's (randomness is keyed by episode).
Prints one JSON object; env G (default 8), EPISODES (1024), MAX_STEPS (1000)."""
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

G = int(os.environ.get("G", "8"))
E = int(os.environ.get("EPISODES", "1024"))
MS = int(os.environ.get("MAX_STEPS", "1000"))
gm = W.CONFIGS["C5"]["map"]()
m = Q.Model(gm, action_mask=W.A9)
m.value_iteration(1e-9)
m.run_episodes(8, max_steps=5, planner=Q.QVTS_PLANNER_QVTS, depth=3, n_samples=8, seed=99)   # warm
torch.cuda.synchronize()
ranks = []
outcomes = np.zeros(4, np.int64)
steps_total = 0
for r in range(G):
    comm = Q.make_callback_comm(r, G, lambda ptr, count, stream: None)
    t0 = time.perf_counter()
    rec, _ = m.run_episodes(E, max_steps=MS, stop_patience=3, planner=Q.QVTS_PLANNER_QVTS, depth=3, n_samples=8,
                            seed=1, comm=comm)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    own = np.arange(E) % G == r
    steps = int(rec["steps"][own].sum())
    steps_total += steps
    for k in range(4):
        outcomes[k] += int((rec["outcome"][own] == k).sum())
    ranks.append({"rank": r, "wall_s": dt, "episodes": int(own.sum()), "episode_steps": steps})
    print(json.dumps(ranks[-1]), file=sys.stderr, flush=True)
worst = max(x["wall_s"] for x in ranks)
print(json.dumps({"config": f"C5: random(256,256,0.2,seed=5), A9, D=3, n=8, {E} episodes, max_steps {MS}, "
                            f"sharded e = r mod {G}, ranks run in turn on one B200",
                  "G": G, "ranks": ranks, "max_rank_wall_s": worst,
                  "mean_rank_wall_s": float(np.mean([x["wall_s"] for x in ranks])),
                  "episode_steps": steps_total, "outcomes": {str(k): int(outcomes[k]) for k in range(4)}}),
      flush=True)
