"""Multi-rank protocol on CPU (world_size 2, gloo): the sharded plan step and the episode-record
reduction of SURVEY §8(e), with the oracle standing in for each rank's subtree work.

Plan step: every rank replicates the levels above the shard level L_s, evaluates the level-L_s
V-nodes it owns (canonical index i ≡ rank mod G, as libqvts does), writes them into a
zero-padded fp64 array, all-reduces it (sum) and backs up to the root — the root Q must equal the
unsharded plan bit for bit.  Episodes: rank r runs e ≡ r (mod G); the summed zero-padded records
equal a single-rank run."""
import os

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle as O
import workloads as W

G = 2
DEPTH, N, SEED, SHARD_MIN = 3, 4, 11, 4


def _setup():
    gm = W.random_map(7, 8, 0.2, seed=21)
    m = O.Model.grid(gm, action_mask=W.A8)
    _, _, Q, _, _ = m.value_iteration(1e-9)
    return gm, m, Q


def _levels(m, Q, b0):
    """Replicated part: the oracle's own tree, V-nodes per level in canonical (parent, a, z)
    order, with each Q-node's R and counts (for the backup above the shard level)."""
    res = m.plan(Q, b0, DEPTH, N, seed=SEED, trace=True, capture_beliefs=True)
    t = res.trace
    qinfo = {int(p): (float(R), cnt.copy()) for p, R, cnt in zip(t.q_path, t.q_R, t.q_cnt)}
    levels = [[(0, b0)]]
    for d in range(DEPTH - 1):
        nxt = []
        for vpath, _ in levels[-1]:
            for a in m.action_ids:
                qp = O.qpath_child(vpath, d, a)
                _, cnt = qinfo[qp]
                for z in range(16):
                    if cnt[z]:
                        cp = O.vpath_child(qp, d, z)
                        nxt.append((cp, t.v_belief[cp]))
        levels.append(nxt)
    return res, qinfo, levels


def _backup(m, qinfo, levels, Vshard, Ls):
    """Back up from the (complete) shard level to the root: Q = R + γ Σ (f/n) V, V = max_a Q."""
    V = {levels[Ls][i][0]: Vshard[i] for i in range(len(levels[Ls]))}
    for d in range(Ls - 1, -1, -1):
        newV = {}
        for vpath, _ in levels[d]:
            qs = []
            for a in m.action_ids:
                qp = O.qpath_child(vpath, d, a)
                R, cnt = qinfo[qp]
                acc = 0.0
                for z in range(16):
                    if cnt[z]:
                        acc += (cnt[z] / N) * V[O.vpath_child(qp, d, z)]
                qs.append(R + 0.95 * acc)
            newV[vpath] = max(qs)
            if d == 0:
                root_q = qs
        V = newV
    return np.array(root_q)


def _worker(rank, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=G)
    try:
        gm, m, Q = _setup()
        b0 = W.uniform_belief(gm)
        ref, qinfo, levels = _levels(m, Q, b0)
        Ls = next(d for d in range(1, DEPTH) if len(levels[d]) >= SHARD_MIN * G)
        nodes = levels[Ls]
        buf = torch.zeros(len(nodes), dtype=torch.float64)
        owned = list(range(rank, len(nodes), G))
        for i in owned:
            vpath, b = nodes[i]
            v, _ = m.vnode_value(Q, b, vpath, Ls, DEPTH, N, seed=SEED)
            buf[i] = v + 0.0
        dist.all_reduce(buf, op=dist.ReduceOp.SUM)
        root_q = _backup(m, qinfo, levels, buf.numpy(), Ls)
        # episodes: e ≡ rank (mod G), zero-padded records summed across ranks
        E = 5
        rec = torch.zeros(E, 4, dtype=torch.float64)
        for e in range(rank, E, G):
            r, _, _, _ = m.run_episode(Q, b0, O.PLANNER_MDP, max_steps=40, seed=3, episode=e)
            rec[e] = torch.tensor([r.outcome, r.steps, r.collisions, r.disc_return], dtype=torch.float64)
        dist.all_reduce(rec, op=dist.ReduceOp.SUM)
        q.put((rank, root_q.tolist(), ref.qroot.tolist(), len(owned), len(nodes), Ls, rec.numpy().tolist()))
    finally:
        dist.destroy_process_group()


def test_sharded_protocol_gloo_world2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + os.getpid() % 1000
    ps = [ctx.Process(target=_worker, args=(r, port, q)) for r in range(G)]
    for p in ps:
        p.start()
    out = [q.get(timeout=240) for _ in range(G)]
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    out.sort()
    owned_total = sum(o[3] for o in out)
    assert owned_total == out[0][4] and out[0][5] >= 1          # every shard-level node owned once
    for rank, root_q, ref_q, *_ in out:
        assert root_q == ref_q, f"rank {rank}: sharded root Q differs from the unsharded plan"
    # episode records identical on both ranks and equal to a single-rank run
    assert out[0][6] == out[1][6]
    gm, m, Q = _setup()
    b0 = W.uniform_belief(gm)
    for e in range(5):
        r, _, _, _ = m.run_episode(Q, b0, O.PLANNER_MDP, max_steps=40, seed=3, episode=e)
        assert out[0][6][e] == [r.outcome, r.steps, r.collisions, r.disc_return]
