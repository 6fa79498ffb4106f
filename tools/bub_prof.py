"""Batched belief update only (for an ncu launch list): C4 map, 2048 beliefs, mixed actions, z = 15."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import workloads as W  # noqa: E402
from paper_1810_00204_b200 import qvts as Q  # noqa: E402

gm = W.CONFIGS["C4"]["map"]()
m = Q.Model(gm, action_mask=W.A8)
NB = 2048
bb = torch.tensor(np.stack([W.random_belief(gm, 500 + i % 64, dtype=np.float32) for i in range(NB)]), device="cuda")
ob = torch.empty_like(bb)
acts = np.array([m.action_ids[i % m.n_actions] for i in range(NB)], np.int32)
zs = np.full(NB, 15, np.int32)
for _ in range(2):
    m.belief_update_batch(bb, acts, zs, ob)
torch.cuda.synchronize()
