"""Context numbers at the paper's Table-I map size (100x40, 9 actions, |Z| = 16, uniform start;
PAPER.md:372, 394): level-batched plan-step latency at depth 3 and 4 (n = 16), and the anytime
best-first planner's time for fixed expansion budgets.  The paper's 1376 ms per step (laptop CPU
+ Maxwell GPU, time budget unknown) is context, not a comparable measurement."""
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

gm = W.paper_style(40, 100, 8, 20, seed=7)
m = Q.Model(gm, action_mask=W.A9)
m.value_iteration()
m.fib_iteration()
b = torch.tensor(W.uniform_belief(gm, np.float32), device="cuda")
Q.qvts_pbvi(m.h, b, 4, 32, 1, 30)
out = {"map": "paper_style(40, 100, 8 walls, 20 pillars, seed 7), A9, uniform b0", "free_cells": int((gm.occupancy == 0).sum())}
for D in (3, 4):
    m.plan_step(b, D, 16, seed=1, step=100)
    lat, upd = [], []
    for k in range(10):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        r = m.plan_step(b, D, 16, seed=1, step=k)
        torch.cuda.synchronize()
        lat.append((time.perf_counter() - t0) * 1e3)
        upd.append(r.n_belief_updates)
    out[f"level_batched_D{D}_n16"] = {"ms_median": float(np.median(lat)), "updates_per_step": float(np.mean(upd))}
for E in (100, 1000, 5000):
    m.plan_best_first(b, 16, E, max_depth=8, seed=1, step=99)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    r = m.plan_best_first(b, 16, E, max_depth=8, seed=1, step=0)
    torch.cuda.synchronize()
    out[f"best_first_E{E}"] = {"ms": (time.perf_counter() - t0) * 1e3, "expansions": r.n_expansions,
                               "vnodes": r.n_vnodes, "U": r.U, "L": r.L, "stop": r.stop_reason}
print(json.dumps(out), flush=True)
