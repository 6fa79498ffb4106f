"""Best-first QVTS (NEXT-2) at the bench workload (C4: 256x256, A8) on one B200: PBVI build time,
then expansions/s of qvts_plan_best_first with per-class kernel times.  Prints one JSON object."""
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

cfgname = os.environ.get("BF_CONFIG", "C4")
gm = W.CONFIGS[cfgname]["map"]()
m = Q.Model(gm, action_mask=W.A8)
b = torch.tensor(W.uniform_belief(gm, np.float32), device="cuda")
out = {"config": cfgname, "cells": m.n_cells}
torch.cuda.synchronize()
t0 = time.perf_counter()
m.fib_iteration(1e-9)
torch.cuda.synchronize()
out["fib_s"] = time.perf_counter() - t0
PTS = int(os.environ.get("BF_POINTS", "32"))
t0 = time.perf_counter()
n_pts = Q.qvts_pbvi(m.h, b, 4, PTS, 1, 30)
torch.cuda.synchronize()
out["pbvi"] = {"s": time.perf_counter() - t0, "points": n_pts, "sweeps": 30}
t0 = time.perf_counter()
n_big = Q.qvts_pbvi(m.h, b, 7, 128, 1, 30)
torch.cuda.synchronize()
out["pbvi_128"] = {"s": time.perf_counter() - t0, "points": n_big, "sweeps": 30, "expansion_rounds": 7}
Q.qvts_pbvi(m.h, b, 4, PTS, 1, 30)   # the set the planner below uses
for n, E in ((16, 50), (16, 400), (16, 2000)):
    m.plan_best_first(b, n, E, max_depth=8, seed=1)        # warm (pool sized, graph path)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    r = m.plan_best_first(b, n, E, max_depth=8, seed=1, step=1)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    rec = {"wall_ms": dt * 1e3, "device_ms": r.device_ms, "expansions": r.n_expansions,
           "expansions_per_s": r.n_expansions / dt, "vnodes": r.n_vnodes, "stop": r.stop_reason, "U": r.U, "L": r.L}
    if E == 400:
        Q.qvts_set_profiling(m.h, True)
        m.plan_best_first(b, n, E, max_depth=8, seed=1, step=1)
        prof = Q.qvts_get_profile(m.h)
        Q.qvts_set_profiling(m.h, False)
        rec["kernel_ms_profiled_run"] = {k: round(v, 2) for k, v in prof["ms"].items()}
    out[f"n{n}_E{E}"] = rec
print(json.dumps(out), flush=True)
