"""The library's own multi-rank path end to end ("parallel samples"):
two processes on the one GPU, `torch.distributed` over gloo, `make_torch_comm` -> the
`allreduce_sum_f64` callback that `qvts_plan_step` / `qvts_run_episodes` re-enter.  Each rank
expands only its share of the shard-level V-nodes (plan) or its episodes e = rank (mod 2); the
exchange is one host-side all-reduce per call (no kernel waits on another process).  The root Q,
the action, the level counts and every episode record must equal a single-rank run bit for bit.
"""
import json
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

_RANK = r'''
import json, os, sys
import numpy as np, torch, torch.distributed as dist
sys.path.insert(0, os.environ["QVTS_ROOT"])
import workloads as W
from paper_1810_00204_b200 import qvts as Q
torch.cuda.set_device(0)
world = int(os.environ.get("WORLD_SIZE", "1"))
if world > 1:
    dist.init_process_group("gloo")
rank = dist.get_rank() if world > 1 else 0
gm = W.CONFIGS["C3"]["map"]()
m = Q.Model(gm, action_mask=W.A8)
m.value_iteration(1e-9)
comm = Q.make_torch_comm(min_nodes_per_rank=4) if world > 1 else None
b = torch.tensor(W.uniform_belief(gm, np.float32), device="cuda")
out = {"plan": []}
for step in (0, 1):
    r = m.plan_step(b, 3, 8, seed=5, step=step, comm=comm)
    out["plan"].append({"q": [float(x).hex() for x in r.q_root[:m.n_actions]], "action": r.action,
                        "nv": list(r.n_vnodes[:4]), "shard_level": r.shard_level})
gm2 = W.random_map(24, 24, 0.2, seed=8)
m2 = Q.Model(gm2, action_mask=W.A9)
m2.value_iteration(1e-9)
comm2 = Q.make_torch_comm(min_nodes_per_rank=4) if world > 1 else None
rec, _ = m2.run_episodes(6, max_steps=25, planner=Q.QVTS_PLANNER_QVTS, depth=2, n_samples=4, seed=3, comm=comm2)
out["episodes"] = {k: [float(x).hex() if isinstance(x, float) else int(x) for x in v.tolist()] for k, v in rec.items()}
out["rank"] = rank
if rank == 0:
    json.dump(out, open(os.environ["QVTS_OUT"], "w"))
if world > 1:
    dist.barrier()
    dist.destroy_process_group()
'''


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _run(tmp_path, world):
    script = tmp_path / "rank.py"
    script.write_text(_RANK)
    out = tmp_path / f"out{world}.json"
    env = dict(os.environ, QVTS_ROOT=ROOT, QVTS_OUT=str(out))
    if world == 1:
        cmd = [sys.executable, str(script)]
    else:
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
               "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), str(script)]
    r = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-4000:]
    return json.loads(out.read_text())


def test_two_processes_gloo_match_one_rank_bitwise(tmp_path):
    one = _run(tmp_path, 1)
    two = _run(tmp_path, 2)
    for a, b in zip(one["plan"], two["plan"]):
        assert a["q"] == b["q"] and a["action"] == b["action"]
        assert a["shard_level"] == -1 and b["shard_level"] >= 1
        # levels above the shard level are replicated; below it each rank holds its share
        assert a["nv"][:b["shard_level"] + 1] == b["nv"][:b["shard_level"] + 1]
    assert one["episodes"] == two["episodes"]
