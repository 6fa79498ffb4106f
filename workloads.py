"""Seeded synthetic inputs shared by the oracle tests, the GPU parity tests and bench.py.

This module holds NO arithmetic of the QVTS method (no transition, observation, reward,
Bayes update, sampling or backup).  It only draws occupancy maps, goal cells and
probability vectors with numpy's seeded generator, with the shapes and structure of the
paper's workloads (recipe restated in DESIGN.md "Input recipe"):

* ``pillars(H, W, k, seed)``   an empty room with k isolated 1-cell obstacles ("landmarks",
  reading R20: sensed only through the paper's 4 wall sensors, §V).
* ``random_map(H, W, rho, seed)``  Bernoulli(rho) obstacles (configs C3/C4/C5).
* ``paper_style(H, W, walls, pillars, seed)``  straight wall segments with 3-cell doorways
  plus pillars, shaped like the paper's 100x40 office map (§V-B, Fig. 4 missing).

Every generator keeps only the largest 4-connected free component (all other free cells
become occupied) and places the goal on a seeded free cell, so every free cell can reach the
goal (reading R21).  Row 0 is the top row; cell index i = r*W + c.
"""
from __future__ import annotations

from collections import deque
from dataclasses import dataclass

import numpy as np


@dataclass(frozen=True)
class GridMap:
    height: int
    width: int
    occupancy: np.ndarray  # uint8 [H*W], 1 = occupied
    goal: int

    @property
    def n_free(self) -> int:
        return int((self.occupancy == 0).sum())


def _largest_component(occ2d: np.ndarray) -> np.ndarray:
    """Label 4-connected free components by BFS; return a boolean mask of the largest
    (ties: the component whose first cell in row-major order comes first)."""
    H, W = occ2d.shape
    label = -np.ones((H, W), dtype=np.int64)
    sizes = []
    for r0 in range(H):
        for c0 in range(W):
            if occ2d[r0, c0] or label[r0, c0] >= 0:
                continue
            lab = len(sizes)
            q = deque([(r0, c0)])
            label[r0, c0] = lab
            n = 0
            while q:
                r, c = q.popleft()
                n += 1
                for dr, dc in ((-1, 0), (1, 0), (0, -1), (0, 1)):
                    rr, cc = r + dr, c + dc
                    if 0 <= rr < H and 0 <= cc < W and not occ2d[rr, cc] and label[rr, cc] < 0:
                        label[rr, cc] = lab
                        q.append((rr, cc))
            sizes.append(n)
    if not sizes:
        raise ValueError("map has no free cell")
    best = int(np.argmax(sizes))
    return label == best


def _finish(occ2d: np.ndarray, rng: np.random.Generator) -> GridMap:
    keep = _largest_component(occ2d)
    occ = np.where(keep, 0, 1).astype(np.uint8)
    free = np.flatnonzero(occ.reshape(-1) == 0)
    goal = int(free[rng.integers(len(free))])
    H, W = occ.shape
    return GridMap(H, W, occ.reshape(-1).copy(), goal)


def pillars(H: int, W: int, k: int, seed: int) -> GridMap:
    """Empty room plus k isolated interior pillar cells (no two pillars 8-adjacent)."""
    rng = np.random.default_rng(seed)
    occ = np.zeros((H, W), dtype=np.uint8)
    placed = 0
    tries = 0
    while placed < k and tries < 100000:
        tries += 1
        r = int(rng.integers(1, max(2, H - 1)))
        c = int(rng.integers(1, max(2, W - 1)))
        if r >= H or c >= W:
            continue
        if occ[max(0, r - 1):r + 2, max(0, c - 1):c + 2].any():
            continue
        occ[r, c] = 1
        placed += 1
    return _finish(occ, rng)


def random_map(H: int, W: int, rho: float, seed: int) -> GridMap:
    """Bernoulli(rho) obstacles."""
    rng = np.random.default_rng(seed)
    occ = (rng.random((H, W)) < rho).astype(np.uint8)
    return _finish(occ, rng)


def paper_style(H: int, W: int, walls: int, n_pillars: int, seed: int) -> GridMap:
    """Straight wall segments of length W/4..W/2 (H/4..H/2 for vertical ones), each with a
    3-cell doorway, plus isolated pillars."""
    rng = np.random.default_rng(seed)
    occ = np.zeros((H, W), dtype=np.uint8)
    for _ in range(walls):
        if rng.random() < 0.5:  # horizontal
            L = int(rng.integers(max(3, W // 4), max(4, W // 2) + 1))
            r = int(rng.integers(1, H - 1))
            c0 = int(rng.integers(0, max(1, W - L)))
            occ[r, c0:c0 + L] = 1
            d = c0 + int(rng.integers(0, max(1, L - 3)))
            occ[r, d:d + 3] = 0
        else:
            L = int(rng.integers(max(3, H // 4), max(4, H // 2) + 1))
            c = int(rng.integers(1, W - 1))
            r0 = int(rng.integers(0, max(1, H - L)))
            occ[r0:r0 + L, c] = 1
            d = r0 + int(rng.integers(0, max(1, L - 3)))
            occ[d:d + 3, c] = 0
    placed = 0
    tries = 0
    while placed < n_pillars and tries < 100000:
        tries += 1
        r = int(rng.integers(1, H - 1))
        c = int(rng.integers(1, W - 1))
        if occ[r - 1:r + 2, c - 1:c + 2].any():
            continue
        occ[r, c] = 1
        placed += 1
    return _finish(occ, rng)


def corridor(L: int, goal_right: bool = True) -> GridMap:
    """1xL open corridor with the goal at one end (closed-form VI pin P5)."""
    occ = np.zeros(L, dtype=np.uint8)
    return GridMap(1, L, occ, L - 1 if goal_right else 0)


def from_ascii(text: str) -> GridMap:
    """'#' occupied, '.' free, 'G' goal (exactly one). No component pruning."""
    rows = [r for r in text.strip("\n").split("\n")]
    H, W = len(rows), len(rows[0])
    if any(len(r) != W for r in rows):
        raise ValueError("NonRectangular")
    occ = np.zeros(H * W, dtype=np.uint8)
    goal = -1
    for r, row in enumerate(rows):
        for c, ch in enumerate(row):
            if ch == "#":
                occ[r * W + c] = 1
            elif ch == "G":
                if goal >= 0:
                    raise ValueError("MultipleGoals")
                goal = r * W + c
    if goal < 0:
        raise ValueError("MissingGoal")
    return GridMap(H, W, occ, goal)


def uniform_belief(m: GridMap, dtype=np.float64) -> np.ndarray:
    """Uniform over free cells (the paper's start condition)."""
    b = (m.occupancy == 0).astype(np.float64)
    return (b / b.sum()).astype(dtype)


def random_belief(m: GridMap, seed: int, sparsity: float = 0.0, dtype=np.float64) -> np.ndarray:
    """Random dense probability vector on free cells (exponential weights), optionally with a
    seeded fraction of free cells set to exactly zero."""
    rng = np.random.default_rng(seed)
    w = rng.exponential(size=m.occupancy.size)
    w[m.occupancy != 0] = 0.0
    if sparsity > 0:
        w[rng.random(w.size) < sparsity] = 0.0
    if w.sum() == 0:
        w[np.flatnonzero(m.occupancy == 0)[0]] = 1.0
    return (w / w.sum()).astype(dtype)


def point_belief(m: GridMap, cell: int, dtype=np.float64) -> np.ndarray:
    b = np.zeros(m.occupancy.size, dtype=np.float64)
    b[cell] = 1.0
    return b.astype(dtype)


def free_cell(m: GridMap, seed: int) -> int:
    rng = np.random.default_rng(seed)
    free = np.flatnonzero(m.occupancy == 0)
    return int(free[rng.integers(len(free))])


# Action sets as stencil-id masks (reading R19).
A9 = 0x1FF
A8 = 0x1EF
A4 = 0x0AA

# BASELINE.json configs.  Model defaults: gamma .95, noise (.8,.1,.05), acc .95.
CONFIGS = {
    "C1": dict(map=lambda: pillars(10, 10, 3, seed=1), action_mask=A4, depth=2, n=4),
    "C2": dict(map=lambda: paper_style(50, 50, 6, 12, seed=1), action_mask=A9, depth=3, n=16),
    "C3": dict(map=lambda: random_map(128, 128, 0.2, seed=3), action_mask=A8, depth=3, n=8),
    "C4": dict(map=lambda: random_map(256, 256, 0.2, seed=4), action_mask=A8, depth=4, n=16),
    "C5": dict(map=lambda: random_map(256, 256, 0.2, seed=5), action_mask=A9, depth=3, n=8),
}
