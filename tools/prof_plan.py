"""Profiling driver: one warm-up + one timed C4 plan step (for ncu launch lists / captures)."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import workloads as W  # noqa: E402
from paper_1810_00204_b200 import qvts as Q  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C4"
c = W.CONFIGS[cfg]
gm = c["map"]()
m = Q.Model(gm, action_mask=c["action_mask"])
m.value_iteration(1e-9)
b = torch.tensor(W.uniform_belief(gm, np.float32), device="cuda")
for k in range(2):
    r = m.plan_step(b, c["depth"], c["n"], seed=1, step=k)
torch.cuda.synchronize()
print(f"{cfg}: {r.n_belief_updates} updates, {r.device_ms:.2f} ms")
