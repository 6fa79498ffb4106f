"""Debug probe for the tensor-core leaf kernel: depth-1 plans (the root is the leaf level), so
P(z|b,a), R(b,a) and Q of the root Q-nodes expose the class bins.  Compares QVTS_LEAF_MMA=1
against the scalar leaf kernel (=0) for uniform, random and point-mass roots."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import workloads as W  # noqa: E402
from paper_1810_00204_b200 import qvts as Q  # noqa: E402


def run(g, b, flag):
    os.environ["QVTS_LEAF_MMA"] = flag
    r = g.plan_step(torch.tensor(b, device="cuda"), 1, 16, seed=3, step=0, want_trace=True)
    t = g.trace(with_draws=True, n_samples=16)
    q = t["levels"][0]["q"]
    return np.array(q["P"]), np.array(q["R"]), np.array(q["Q"])


def main():
    maps = {"C1": (W.CONFIGS["C1"]["map"](), W.A4), "ragged": (W.random_map(29, 37, 0.2, seed=9), W.A8),
            "C3": (W.CONFIGS["C3"]["map"](), W.A8)}
    for name, (gm, mask) in maps.items():
        g = Q.Model(gm, action_mask=mask)
        g.value_iteration(1e-9)
        free = np.flatnonzero(~np.asarray(gm.occ, bool).ravel()) if hasattr(gm, "occ") else None
        beliefs = {"uniform": W.uniform_belief(gm, np.float32), "random": W.random_belief(gm, 3).astype(np.float32)}
        cells = np.flatnonzero(W.uniform_belief(gm) > 0)
        for c in cells[:: max(1, len(cells) // 6)][:6]:
            beliefs[f"point{c}"] = W.point_belief(gm, int(c)).astype(np.float32)
        for bn, b in beliefs.items():
            P1, R1, Q1 = run(g, b, "1")
            P0, R0, Q0 = run(g, b, "0")
            print(f"{name:7s} {bn:12s} |dP| {np.max(np.abs(P1 - P0)):.2e} |dR| {np.max(np.abs(R1 - R0)):.2e} "
                  f"|dQ| {np.max(np.abs(Q1 - Q0)):.2e}  sumP {P1.sum(1)[:3]} vs {P0.sum(1)[:3]}", flush=True)
            if np.max(np.abs(P1 - P0)) > 1e-5 and bn.startswith("point"):
                print("   P mma  ", np.round(P1[0], 4))
                print("   P ref  ", np.round(P0[0], 4))
                print("   R", R1, R0)
        g.close()


if __name__ == "__main__" and not os.environ.get("LM_DEPTH2"):
    main()


def depth2():
    for name, (gm, mask) in {"C1": (W.CONFIGS["C1"]["map"](), W.A4),
                             "ragged": (W.random_map(29, 37, 0.2, seed=9), W.A8)}.items():
        g = Q.Model(gm, action_mask=mask)
        g.value_iteration(1e-9)
        b = W.random_belief(gm, 3).astype(np.float32)
        res = {}
        for flag in ("1", "0"):
            for graph in ("0", "1"):
                os.environ["QVTS_LEAF_MMA"] = flag
                os.environ["QVTS_PLAN_GRAPH"] = graph
                g.plan_step(torch.tensor(b, device="cuda"), 2, 4, seed=3, step=0, want_trace=True)
                t = g.trace(with_draws=True, n_samples=4)
                q = t["levels"][1]["q"]
                res[flag + graph] = (np.array(q["P"]), np.array(q["R"]))
        NA = g.n_actions
        for k in ("10", "11", "01"):
            dP = np.abs(res[k][0] - res["00"][0]).max(1).reshape(-1, NA).max(1)
            dR = np.abs(res[k][1] - res["00"][1]).reshape(-1, NA).max(1)
            print(name, "mma,graph=" + k, "per-parent max|dP|", np.array2string(dP, precision=1), "max|dR|",
                  np.array2string(dR, precision=1))
        g.close()


if __name__ == "__main__" and os.environ.get("LM_DEPTH2"):
    depth2()
