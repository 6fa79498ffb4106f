"""bench.py — QVTS plan-step throughput on B200 (BASELINE.json metric: belief-node updates/s and
plan-step latency).  Workload (N=1 and every N): config C4 — 256x256 Bernoulli(0.2) map, 8
actions, depth 4, 16 sampled observations per Q-node, uniform root belief.
One step = one full plan step (all S1-S6 rows) on a fresh step key; the tree (≈37 GB of beliefs)
is far larger than L2, so no extra flush is needed between steps.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference]

N>1 runs under torchrun, one rank per GPU: subtrees below the shard level are split across
ranks and finished by one NCCL all-reduce of the shard-level values; time is the
max over ranks.  --impl reference times the fp64 CPU oracle (the deliberately slow reference
arm) on bounded samples of the same workload.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
import workloads as W  # noqa: E402

METRIC = "belief-node updates/sec and QVTS plan-step latency (ms) at 1/2/4/8 B200"
UNIT = "belief-node updates/s"
CFG_NAME = "C4"


def workload_config():
    c = W.CONFIGS[CFG_NAME]
    return c["map"](), c["action_mask"], c["depth"], c["n"]


def config_json(n_gpus, extra=None):
    d = {"workload": "C4: 256x256 random map rho=0.2 (seed 4), A8, depth 4, n=16 samples/Q-node, uniform root",
         "grid": "256x256", "actions": 8, "depth": 4, "n_samples": 16, "gamma": 0.95,
         "noise": [0.8, 0.1, 0.05], "sensor_acc": 0.95,
         "l2_flush": "none needed: inputs larger than L2 (each step writes/reads a ~37 GB belief tree)",
         "parallelism": f"subtree-shard x{n_gpus}" if n_gpus > 1 else "single GPU"}
    if extra:
        d.update(extra)
    return d


# ---- oracle sample (cpu_baseline / --impl reference) --------------------------------------------
def _oracle_setup():
    import oracle as O
    gm, mask, D, n = workload_config()
    om = O.Model.grid(gm, action_mask=mask)
    _, _, Qo, _, _ = om.value_iteration(1e-9)
    return O, gm, om, Qo, D, n


def _oracle_sample(O, gm, om, Qo, D, n, rng, seed=1, step=0):
    """One bounded sample of the workload: follow a random root-to-level-(D-1) path of the
    oracle's own tree, then expand that V-node's full subtree (its |A| Q-nodes and their
    sampled leaves).  Returns the belief-node updates performed."""
    b = W.uniform_belief(gm)
    vpath, updates = 0, 0
    for d in range(D - 1):
        ai = int(rng.integers(om.na))
        qpath = O.qpath_child(vpath, d, om.action_ids[ai])
        P, R, z, flag, cnt = om.qnode_sample(b, ai, qpath, n, seed=seed, step=step)
        zs = np.flatnonzero(cnt)
        zz = int(zs[rng.integers(len(zs))])
        b, _ = om.belief_update(b, ai, zz)
        vpath = O.vpath_child(qpath, d, zz)
        updates += 1
    V, qv = om.vnode_value(Qo, b, vpath, D - 1, D, n, seed=seed, step=step)
    # leaves of the expanded subtree = unique draws of its |A| Q-nodes
    for ai, a in enumerate(om.action_ids):
        _, _, _, _, cnt = om.qnode_sample(b, ai, O.qpath_child(vpath, D - 1, a), n, seed=seed, step=step)
        updates += int((cnt > 0).sum())
    return updates


_ORACLE = None     # set before forking the all-core workers (they share the compiled model)


def _oracle_worker(job):
    """One worker process: bounded oracle samples for budget_s seconds (or `count` samples)."""
    seed, budget_s, count = job
    os.environ["OMP_NUM_THREADS"] = "1"
    O, gm, om, Qo, D, n = _ORACLE
    rng = np.random.default_rng(1000 + seed)
    t0 = time.perf_counter()
    upd, k = 0, 0
    while (count and k < count) or (not count and time.perf_counter() - t0 < budget_s):
        upd += _oracle_sample(O, gm, om, Qo, D, n, rng, step=seed * 100000 + k)
        k += 1
    return upd, k


def _oracle_pool():
    import multiprocessing as mp
    cores = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else (os.cpu_count() or 1)
    return mp.get_context("fork").Pool(cores), cores


def cpu_baseline(budget_s=10.0):
    """the oracle as it stands, single thread and on all of the host's cores
    (one forked worker per core running independent bounded samples of the same workload)."""
    global _ORACLE
    _ORACLE = _oracle_setup()
    t0 = time.perf_counter()
    upd1, k1 = _oracle_worker((0, budget_s, 0))
    dt1 = time.perf_counter() - t0
    pool, cores = _oracle_pool()
    try:
        t0 = time.perf_counter()
        res = pool.map(_oracle_worker, [(1 + i, budget_s, 0) for i in range(cores)])
        dtc = time.perf_counter() - t0
    finally:
        pool.close()
        pool.join()
    updc, kc = sum(r[0] for r in res), sum(r[1] for r in res)
    return {"value": updc / dtc, "unit": UNIT, "cores": cores, "kind": "oracle",
            "sample": f"{kc} level-3 subtrees of the C4 depth-4 tree (oracle's own random paths, all 8 actions and "
                      f"sampled leaves each) on {cores} worker processes, {updc} belief-node updates in {dtc:.1f} s, "
                      f"fp64",
            "single_thread": {"value": upd1 / dt1, "cores": 1,
                              "sample": f"{k1} subtrees, {upd1} updates in {dt1:.1f} s"}}


def run_reference(args):
    """--impl reference: the oracle on all host cores; each step = one bounded sample per core."""
    global _ORACLE
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    _ORACLE = _oracle_setup()
    pool, cores = _oracle_pool()
    try:
        for i in range(args.warmup):
            pool.map(_oracle_worker, [(10000 * (i + 1) + c, 0.0, 1) for c in range(cores)])
        t0 = time.perf_counter()
        upd = 0
        for i in range(args.steps):
            res = pool.map(_oracle_worker, [(10000 * (args.warmup + i + 1) + c, 0.0, 1) for c in range(cores)])
            upd += sum(r[0] for r in res)
        dt = time.perf_counter() - t0
    finally:
        pool.close()
        pool.join()
    v = upd / dt
    line = {"metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * dt / max(1, args.steps), "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic", "impl": "reference",
            "config": config_json(1, {"step": f"one bounded sample per host core: {cores} random level-3 V-node "
                                              f"subtrees of the C4 tree"}),
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": cores, "kind": "oracle",
                             "sample": f"{args.steps} steps x {cores} level-3 subtrees of the C4 depth-4 tree, "
                                       f"{upd} updates"},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ---- clocks ------------------------------------------------------------------------------------
class ClockSampler:
    Q = ("index,clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.p = None

    def __enter__(self):
        try:
            self.p = subprocess.Popen(["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}",
                                       "--format=csv,noheader,nounits", "-lms", "200"],
                                      stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.p = None
        return self

    def __exit__(self, *a):
        self.rows = []
        if self.p is None:
            return
        self.p.terminate()
        out, _ = self.p.communicate(timeout=10)
        for line in out.strip().splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) >= 8:
                self.rows.append(f)

    def summary(self):
        if not getattr(self, "rows", None):
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if r[4 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


# ---- our arm -----------------------------------------------------------------------------------
# Algorithmic FP32 work of S1+S2+S5 per (leaf parent, free cell): SURVEY §8(d) d.3 counts
# |A| (5 + |A|) + |A| FMA per cell (per action a 4-FMA predict and the class-bin add, |A| products
# b'(y) Q(y, a') into the signature bins, and |A| for R(b,a)) = 112 FMA = 224 flops at A8.  The
# kernel does fewer operations than this (the linear fields of reading B3); the roofline is the
# algorithmic count over the measured time.
FLOPS_PER_LEAF_CELL = {na: 2 * (na * (5 + na) + na) for na in (4, 8, 9)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args)
        return

    import torch
    import torch.distributed as dist
    from paper_1810_00204_b200 import qvts as Q

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # one rank per GPU; QVTS_BENCH_BACKEND=gloo lets several ranks share a GPU to exercise the
    # multi-rank path (the exchange is a host-side all-reduce, no kernel waits on another rank)
    backend = os.environ.get("QVTS_BENCH_BACKEND", "nccl")
    local = local % torch.cuda.device_count()
    torch.cuda.set_device(local)
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)

    cpu_base = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu_base = cpu_baseline()

    gm, mask, D, n = workload_config()
    model = Q.Model(gm, action_mask=mask, device=local)
    code, sweeps, res = model.value_iteration(1e-9)
    assert code == 0, "value iteration did not converge"
    b_host = torch.from_numpy(W.uniform_belief(gm, np.float32)).pin_memory()
    root = b_host.to("cuda", non_blocking=True)
    comm = Q.make_torch_comm(min_nodes_per_rank=16) if world > 1 else None
    stream = torch.cuda.current_stream()

    flagged = []

    def step(k, root_buf):
        r = model.plan_step(root_buf, D, n, seed=1, step=k, comm=comm)
        flagged.append(r.n_flag_candidates)
        upd = [r.n_vnodes[d] for d in range(1, D + 1)]
        sl = r.shard_level
        repl = sum(upd[:sl]) if sl >= 0 else 0          # levels 1..sl are replicated on every rank
        local_upd = sum(upd[sl:]) if sl >= 0 else sum(upd)
        return r, repl, local_upd

    for i in range(args.warmup):
        step(i, root)
    torch.cuda.synchronize()

    # ---- device-timed region: inputs resident in HBM ----
    Q.qvts_set_profiling(model.h, True)
    repl_tot, local_tot = 0, 0
    lat = []
    with ClockSampler(local) as clk:
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for i in range(args.steps):
            r, repl, loc = step(args.warmup + i, root)
            repl_tot += repl
            local_tot += loc
            lat.append(r.device_ms)
        e1.record(stream)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
    ms = e0.elapsed_time(e1)
    prof = Q.qvts_get_profile(model.h)
    Q.qvts_set_profiling(model.h, False)
    if world > 1:
        tdev = "cuda" if backend == "nccl" else "cpu"
        t = torch.tensor([ms], device=tdev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
        u = torch.tensor([float(local_tot)], device=tdev, dtype=torch.float64)
        dist.all_reduce(u, op=dist.ReduceOp.SUM)
        local_tot = u.item()
    total_updates = repl_tot + local_tot
    value = total_updates / (ms / 1e3)

    # ---- end-to-end through the public API with host buffers ----
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    e2e_repl, e2e_loc = 0, 0
    e0.record(stream)
    for i in range(args.steps):
        root.copy_(b_host, non_blocking=True)                 # H2D of the step's input
        r, repl, loc = step(10_000 + i, root)                 # returns host q_root/action (D2H)
        e2e_repl += repl
        e2e_loc += loc
    e1.record(stream)
    torch.cuda.synchronize()
    e2e_ms = e0.elapsed_time(e1)
    if world > 1:
        tdev = "cuda" if backend == "nccl" else "cpu"
        t = torch.tensor([e2e_ms], device=tdev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_ms = float(t.item())
        u = torch.tensor([float(e2e_loc)], device=tdev, dtype=torch.float64)
        dist.all_reduce(u, op=dist.ReduceOp.SUM)
        e2e_loc = u.item()
    e2e_value = (e2e_repl + e2e_loc) / (e2e_ms / 1e3)

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return

    # ---- roofline of the dominant kernel (leaf hist: FP32-ALU bound, SURVEY d.3) ----
    na = model.n_actions
    leaf_ms = prof["ms"]["hist_leaf"]
    leaf_launches = max(1, prof["launches"]["hist_leaf"])
    flops = prof["leaf_cells"] * FLOPS_PER_LEAF_CELL[na]
    achieved = flops / (leaf_ms / 1e3) / 1e12 if leaf_ms > 0 else 0.0
    clocks = clk.summary()
    f_mhz = 1965.0
    peak = 148 * 128 * 2 * f_mhz * 1e6 / 1e12     # FP32 FMA lanes x 2 flops x max SM clock
    share = {k: round(v / max(1e-9, sum(prof["ms"].values())), 4) for k, v in prof["ms"].items()}
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "r02_roofline_traffic.json")
    if os.path.exists(tpath) and CFG_NAME == "C4":
        t = json.load(open(tpath))
        traffic = t["dram_bytes_read"] + t["dram_bytes_write"]
    # ---- the HBM-bound belief kernel (k_correct, S4: child beliefs written once; north star: >= 60%
    # of HBM bandwidth in the belief kernels): algorithmic bytes = 4 * cells per child written
    # (parent reads come through L2), all its launches in the timed region
    corr_ms = prof["ms"]["correct"]
    corr_bytes = 4.0 * prof["correct_cells_written"]
    corr_gbs = corr_bytes / (corr_ms / 1e3) / 1e9 if corr_ms > 0 else 0.0
    peaks = {}
    ppath = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(ppath):
        peaks = json.load(open(ppath))
    copy_peak = float(peaks.get("hbm_gbs", 6549.1))
    wpath = os.path.join(ROOT, "profiles", "r01_hbm_write_peak.json")
    write_peak = json.load(open(wpath))["write_fill"]["GBps"] if os.path.exists(wpath) else None
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f32 beliefs / f64 node scalars", "data": "synthetic",
        "config": config_json(world, {"plan_step_latency_ms_median": statistics.median(lat),
                                      "belief_updates_per_step": total_updates / args.steps,
                                      "flagged_draws_per_step": statistics.median(flagged[args.warmup:args.warmup + args.steps]),
                                      "vi_sweeps": sweeps,
                                      "instrumentation": "per-launch CUDA events (qvts_set_profiling) stay on in "
                                                         "the timed region; ~1 us per launch, < 0.1% of a step"}),
        "roofline": {"bound": "alu", "kernel": "k_leaf<A8> (leaf level: S1+S2+S5)", "achieved": achieved,
                     "peak": peak, "unit": "TFLOP/s", "frac": achieved / peak if peak else None,
                     "traffic": traffic, "traffic_unit": "bytes per launch (ncu dram__bytes_read+write)",
                     "algorithmic": f"{FLOPS_PER_LEAF_CELL[na]} FP32 flops (FMA = 2) per (leaf parent, free cell) x "
                                    f"{prof['leaf_cells'] / leaf_launches:.3e} per launch; "
                                    "peak = 148 SM x 128 FP32 lanes x 2 x 1965 MHz (guide unit counts)",
                     "avg_launch_ms": leaf_ms / leaf_launches},
        "roofline_hbm": {"bound": "hbm", "kernel": "k_correct (S4 Bayes correction, child beliefs written)",
                         "achieved": corr_gbs, "peak": copy_peak, "unit": "GB/s",
                         "frac": corr_gbs / copy_peak if copy_peak else None,
                         "frac_of_write_peak": (corr_gbs / write_peak) if write_peak else None,
                         "frac_of_8tbs": corr_gbs / 8000.0,
                         "algorithmic": f"4 B x {prof['correct_cells_written'] / max(1, prof['launches']['correct']):.3e}"
                                        " child cells written per launch (parents via L2); peak = MEASURED_PEAKS "
                                        "hbm_gbs (copy), also vs the measured pure-write peak and 8 TB/s",
                         "launches": prof["launches"]["correct"], "total_ms": corr_ms},
        "kernel_share": share,
        "kernel_ms": {k: round(v, 3) for k, v in prof["ms"].items()},
        "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": 4 * model.n_cells,
                "d2h_bytes_per_step": 8 * na + 8 * (D + 1)},
        "gpu_launches": prof["total_launches"],
        "clocks": clocks,
        "cpu_baseline": cpu_base,
    }
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
