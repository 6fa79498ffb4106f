"""Short best-first run for an ncu launch list (kernel durations without host gaps)."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import workloads as W  # noqa: E402
from paper_1810_00204_b200 import qvts as Q  # noqa: E402

gm = W.CONFIGS[os.environ.get("BF_CONFIG", "C4")]["map"]()
m = Q.Model(gm, action_mask=W.A8)
b = torch.tensor(W.uniform_belief(gm, np.float32), device="cuda")
m.fib_iteration(1e-9)
Q.qvts_pbvi(m.h, b, 4, 32, 1, 30)
r = m.plan_best_first(b, 16, int(os.environ.get("BF_E", "20")), max_depth=8, seed=1, step=1)
torch.cuda.synchronize()
print("expansions", r.n_expansions, "vnodes", r.n_vnodes, "device_ms", r.device_ms)
