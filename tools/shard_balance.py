"""Projected strong scaling of the sharded C4 plan step from one GPU: each rank's
share (the replicated levels above the shard level plus its round-robin subtrees) is run in turn
and timed on the device; the projected G-GPU step time is the slowest rank plus the one
latency-bound all-reduce, so speedup(G) = T(1) / max_r T_r.  The exchange is replaced by a
callback that leaves the zero-padded shard values as they are (this rank's values only), which
changes only the backup above the shard level, not the work.  Prints one JSON object."""
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import workloads as W  # noqa: E402
from paper_1810_00204_b200 import qvts as Q  # noqa: E402

cfg = W.CONFIGS["C4"]
gm = cfg["map"]()
m = Q.Model(gm, action_mask=cfg["action_mask"])
m.value_iteration(1e-9)
b = torch.tensor(W.uniform_belief(gm, np.float32), device="cuda")
D, n = cfg["depth"], cfg["n"]
steps = (3, 4, 5)


def timed(step, comm=None):
    r = m.plan_step(b, D, n, seed=1, step=step, comm=comm)
    return r.device_ms, sum(r.n_vnodes[1:D + 1]), r.shard_level


for s in steps:                      # warm: workspace, allocations
    timed(s)
out = {"config": "C4 plan step (random 256x256 rho 0.2, A8, D=4, n=16, uniform root), steps 3..5",
       "single": {}, "sharded": {}}
t1 = [timed(s)[0] for s in steps]
out["single"] = {"ms": [round(x, 3) for x in t1], "ms_mean": float(np.mean(t1))}
for G in (2, 4, 8):
    per_rank = []
    for r in range(G):
        comm = Q.make_callback_comm(r, G, lambda ptr, count, stream: None, min_nodes_per_rank=16)
        ts = [timed(s, comm) for s in steps]
        per_rank.append({"rank": r, "ms_mean": float(np.mean([t[0] for t in ts])),
                         "updates_mean": float(np.mean([t[1] for t in ts])), "shard_level": ts[0][2]})
    worst = max(p["ms_mean"] for p in per_rank)
    out["sharded"][str(G)] = {
        "shard_level": per_rank[0]["shard_level"],
        "rank_ms": [round(p["ms_mean"], 3) for p in per_rank],
        "max_ms": worst, "mean_ms": float(np.mean([p["ms_mean"] for p in per_rank])),
        "imbalance": worst / float(np.mean([p["ms_mean"] for p in per_rank])),
        "projected_speedup": out["single"]["ms_mean"] / worst,
        "projected_efficiency": out["single"]["ms_mean"] / worst / G,
    }
print(json.dumps(out), flush=True)
