"""Per-row measurements beside bench.py's plan-step line (one B200): S7 value iteration, NEXT-1
FIB iteration, the qvts_belief_update ABI call (S1+S2+S4 on one Q-node), the leaf bound swap,
and a bounded C5-style episode batch (S8).  Prints one JSON object."""
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


def timed(fn, reps=1):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        out = fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / reps, out


out = {}
gm = W.CONFIGS["C4"]["map"]()
m = Q.Model(gm, action_mask=W.A8)
m.value_iteration(1e-9)                                     # first call: module load, workspace
m.fib_iteration(1e-9)
dt, (code, sw, res) = timed(lambda: m.value_iteration(1e-9))
out["S7_value_iteration_C4"] = {"ms": dt * 1e3, "sweeps": sw, "residual": res, "cells": m.n_cells}
dt, (code, sw, res) = timed(lambda: m.fib_iteration(1e-9))
out["NEXT1_fib_iteration_C4"] = {"ms": dt * 1e3, "sweeps": sw, "residual": res,
                                 "dfma_per_sweep": m.n_cells * m.n_actions * 16 * m.n_actions * 4}
b = torch.tensor(W.uniform_belief(gm, np.float32), device="cuda")
o = torch.empty_like(b)
m.belief_update(b, 1, 0, o)
dt, p = timed(lambda: m.belief_update(b, 1, 0, o), reps=50)
out["K9_belief_update_C4"] = {"us_per_call": dt * 1e6, "algorithmic_bytes": 8 * m.n_cells,
                              "effective_GBps": 8 * m.n_cells / dt / 1e9,
                              "note": "synchronous ABI call (the batched path with n = 1: one cluster pass + P readback)"}
# batched Eq. 3 (K9 at HBM scale): n beliefs read, n posteriors written
NB = 2048
bb = torch.tensor(np.stack([W.random_belief(gm, 500 + i % 64, dtype=np.float32) for i in range(NB)]), device="cuda")
ob = torch.empty_like(bb)
acts = np.array([m.action_ids[i % m.n_actions] for i in range(NB)], np.int32)
zs = np.full(NB, 15, np.int32)
m.belief_update_batch(bb, acts, zs, ob)
dt, _ = timed(lambda: m.belief_update_batch(bb, acts, zs, ob), reps=5)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
m.belief_update_batch(bb, acts, zs, ob)
e1.record()
torch.cuda.synchronize()
dev_ms = e0.elapsed_time(e1)
out["K9_belief_update_batch_C4"] = {"n": NB, "ms_per_batch": dt * 1e3, "device_ms": dev_ms,
                                    "algorithmic_bytes": NB * 8 * m.n_cells,
                                    "effective_GBps": NB * 8 * m.n_cells / dt / 1e9,
                                    "effective_GBps_device": NB * 8 * m.n_cells / (dev_ms / 1e3) / 1e9,
                                    "note": "read b + write b' per pair (algorithmic); one pass per belief on a thread-block cluster (k_bu_cluster: staged rows, normaliser parts summed through DSMEM, posterior written), one sync"}
# the two-pass path (QVTS_BU_CLUSTER=0), for comparison
os.environ["QVTS_BU_CLUSTER"] = "0"
m.belief_update_batch(bb, acts, zs, ob)
e0.record()
m.belief_update_batch(bb, acts, zs, ob)
e1.record()
torch.cuda.synchronize()
dev2 = e0.elapsed_time(e1)
os.environ.pop("QVTS_BU_CLUSTER")
out["K9_belief_update_batch_C4"]["two_pass_device_ms"] = dev2
out["K9_belief_update_batch_C4"]["two_pass_effective_GBps_device"] = NB * 8 * m.n_cells / (dev2 / 1e3) / 1e9
for leaf in (Q.QVTS_LEAF_QMDP, Q.QVTS_LEAF_FIB):
    m.plan_step(b, 4, 16, seed=1, step=0, leaf_bound=leaf)
    dt, r = timed(lambda: m.plan_step(b, 4, 16, seed=1, step=1, leaf_bound=leaf), reps=3)
    out[f"plan_C4_leaf_{'fib' if leaf else 'qmdp'}"] = {"ms": dt * 1e3, "updates": r.n_belief_updates,
                                                         "updates_per_s": r.n_belief_updates / dt}
m.plan_step(b, 4, 16, seed=1, step=0, sampler=Q.QVTS_SAMPLER_ANCESTRAL)
dt, r = timed(lambda: m.plan_step(b, 4, 16, seed=1, step=1, sampler=Q.QVTS_SAMPLER_ANCESTRAL), reps=3)
out["NEXT3_plan_C4_ancestral_sampler"] = {"ms": dt * 1e3, "updates": r.n_belief_updates,
                                          "updates_per_s": r.n_belief_updates / dt}
m.close()

E = int(os.environ.get("EPISODES", "128"))
MS = int(os.environ.get("MAX_STEPS", "100"))
gm5 = W.CONFIGS["C5"]["map"]()
m5 = Q.Model(gm5, action_mask=W.A9)
m5.value_iteration(1e-9)
Q.qvts_set_profiling(m5.h, True)
dt, (rec, _) = timed(lambda: m5.run_episodes(E, max_steps=MS, stop_patience=3, planner=0, depth=3, n_samples=8, seed=1))
prof = Q.qvts_get_profile(m5.h)
steps = int(rec["steps"].sum())
out["S8_episodes_C5_bounded"] = {"episodes": E, "max_steps": MS, "wall_s": dt, "episode_steps": steps,
                                 "episode_steps_per_s": steps / dt,
                                 "outcomes": {str(k): int((rec["outcome"] == k).sum()) for k in range(4)},
                                 "kernel_ms": {k: round(v, 1) for k, v in prof["ms"].items()},
                                 "config": "C5 map random(256,256,0.2,seed 5), A9, D=3, n=8, uniform b0"}
print(json.dumps(out), flush=True)
