"""Small-config exercise of every library entry point (for compute-sanitizer memcheck)."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import workloads as W  # noqa: E402
from paper_1810_00204_b200 import qvts as Q  # noqa: E402

for gm, mask in ((W.CONFIGS["C1"]["map"](), W.A4), (W.random_map(13, 17, 0.2, seed=2), W.A8),
                 (W.paper_style(30, 30, 3, 5, seed=1), W.A9)):
    m = Q.Model(gm, action_mask=mask)
    m.value_iteration(1e-9)
    m.fib_iteration(1e-9)
    b = torch.tensor(W.uniform_belief(gm, np.float32), device="cuda")
    out = torch.empty_like(b)
    m.belief_update(b, m.action_ids[0], 3, out)
    for leaf in (0, 1):
        for sampler in (0, 1):
            m.plan_step(b, 2, 8, seed=1, want_trace=True, leaf_bound=leaf, sampler=sampler)
            m.trace(with_draws=True, n_samples=8, beliefs=True)
    m.plan_step(b, 3, 4, seed=2)
    for pl in (0, 1, 2):
        m.run_episodes(3, max_steps=12, planner=pl, depth=2, n_samples=4, seed=1)
    m.close()
torch.cuda.synchronize()
print("sanitize_small ok")
