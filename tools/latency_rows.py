"""SURVEY §8(d) d.1 rows beside bench.py: C3 plan-step latency (median, p90 over 20 step keys)
and updates/s; C4 density sensitivity (rho 0.1 / 0.3, 5 step keys each).  CUDA events on the
launching stream around each qvts_plan_step.  Prints one JSON object."""
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import workloads as W  # noqa: E402
from paper_1810_00204_b200 import qvts as Q  # noqa: E402


def run(gm, mask, depth, n, keys):
    m = Q.Model(gm, action_mask=mask)
    m.value_iteration(1e-9)
    b = torch.tensor(W.uniform_belief(gm, np.float32), device="cuda")
    for k in keys:                                          # warm: workspace sized for every key
        m.plan_step(b, depth, n, seed=1, step=k)
    st = torch.cuda.current_stream()
    lat, upd = [], []
    for k in keys:
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record(st)
        r = m.plan_step(b, depth, n, seed=1, step=k)
        e1.record(st)
        torch.cuda.synchronize()
        lat.append(e0.elapsed_time(e1))
        upd.append(r.n_belief_updates)
    m.close()
    lat = np.array(lat)
    ups = float(np.sum(upd) / (lat.sum() / 1e3))
    return {"latency_ms_median": float(np.median(lat)), "latency_ms_p90": float(np.percentile(lat, 90)),
            "latency_ms_max": float(lat.max()), "updates_per_step_mean": float(np.mean(upd)), "updates_per_s": ups,
            "cell_updates_per_s": ups * gm.occupancy.size, "keys": len(keys)}


out = {}
c3 = W.CONFIGS["C3"]
out["C3"] = run(c3["map"](), c3["action_mask"], c3["depth"], c3["n"], range(20))
out["C3"]["config"] = "random(128,128,0.2,seed=3), A8, D=3, n=8, uniform root, steps 0..19"
for rho in (0.1, 0.3):
    out[f"C4_rho{rho}"] = run(W.random_map(256, 256, rho, seed=4), W.A8, 4, 16, range(5))
    out[f"C4_rho{rho}"]["config"] = f"random(256,256,{rho},seed=4), A8, D=4, n=16, uniform root, steps 0..4"
print(json.dumps(out), flush=True)
