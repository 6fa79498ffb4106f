"""A/B of the leaf-level split (QVTS_LEAF_NSPLIT) and the leaf kernel (QVTS_LEAF_KERNEL), set in the
environment by the caller: C3 plan-step latency (median of 10 step keys, CUDA events) and a bounded
C5 episode batch (EPISODES x MAX_STEPS, wall clock).  Prints one JSON object."""
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

out = {"QVTS_LEAF_NSPLIT": os.environ.get("QVTS_LEAF_NSPLIT"), "QVTS_LEAF_KERNEL": os.environ.get("QVTS_LEAF_KERNEL")}
c3 = W.CONFIGS["C3"]
gm = c3["map"]()
m = Q.Model(gm, action_mask=c3["action_mask"])
m.value_iteration(1e-9)
b = torch.tensor(W.uniform_belief(gm, np.float32), device="cuda")
for k in range(10):
    m.plan_step(b, 3, 8, seed=1, step=k)
st = torch.cuda.current_stream()
lat = []
for k in range(10):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(st)
    m.plan_step(b, 3, 8, seed=1, step=k)
    e1.record(st)
    torch.cuda.synchronize()
    lat.append(e0.elapsed_time(e1))
out["C3_latency_ms_median"] = float(np.median(lat))
m.close()
E = int(os.environ.get("EPISODES", "128"))
MS = int(os.environ.get("MAX_STEPS", "200"))
gm = W.CONFIGS["C5"]["map"]()
m = Q.Model(gm, action_mask=W.A9)
m.value_iteration(1e-9)
m.run_episodes(8, max_steps=5, planner=Q.QVTS_PLANNER_QVTS, depth=3, n_samples=8, seed=99)
torch.cuda.synchronize()
t0 = time.perf_counter()
rec, _ = m.run_episodes(E, max_steps=MS, stop_patience=3, planner=Q.QVTS_PLANNER_QVTS, depth=3, n_samples=8, seed=1)
torch.cuda.synchronize()
dt = time.perf_counter() - t0
out["C5_episodes"] = E
out["C5_wall_s"] = dt
out["C5_steps_per_s"] = float(rec["steps"].sum()) / dt
print(json.dumps(out), flush=True)
