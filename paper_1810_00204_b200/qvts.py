"""Thin ctypes binding of libqvts.so (include/qvts.h).  Argument marshalling only: every step of
the QVTS path runs in the library's sm_100a kernels.  PyTorch is used for device memory,
streams and torch.distributed; there is no CPU fallback — loading fails loudly when the CUDA
library is missing.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("QVTS_LIB") or os.path.join(_HERE, "libqvts.so")   # QVTS_LIB: A/B builds

QVTS_OK = 0
STATUS = {0: "OK", 1: "INVALID_ARG", 2: "INVALID_MODEL", 3: "STATE", 4: "NOT_CONVERGED",
          5: "ZERO_LIKELIHOOD", 6: "OUT_OF_MEMORY", 7: "CUDA", 8: "COMM"}
QVTS_PLANNER_QVTS, QVTS_PLANNER_MDP, QVTS_PLANNER_ASTAR = 0, 1, 2

# Symbols include/qvts.h declares (checked by tests/test_abi.py).
EXPORTS = [
    "qvts_model_create", "qvts_model_destroy", "qvts_last_error", "qvts_model_info", "qvts_model_tables",
    "qvts_value_iteration", "qvts_get_q", "qvts_belief_update", "qvts_plan_step", "qvts_trace_qnodes",
    "qvts_trace_vnodes", "qvts_trace_leaf_values", "qvts_trace_belief", "qvts_run_episodes",
    "qvts_trace_counts", "qvts_set_profiling", "qvts_get_profile", "qvts_fib_iteration", "qvts_get_alpha",
    "qvts_pbvi", "qvts_get_pbvi", "qvts_plan_best_first", "qvts_trace_best_first", "qvts_bf_advance", "qvts_belief_update_batch",
    "qvts_trace_state_draws",
]
QVTS_BF_BUDGET, QVTS_BF_GAP, QVTS_BF_TERMINAL, QVTS_BF_POOL, QVTS_BF_TIME = 0, 1, 2, 3, 4
QVTS_LEAF_QMDP, QVTS_LEAF_FIB = 0, 1
QVTS_SAMPLER_MARGINAL, QVTS_SAMPLER_ANCESTRAL = 0, 1


class QvtsError(RuntimeError):
    def __init__(self, code: int, where: str, msg: str):
        super().__init__(f"{where}: {STATUS.get(code, code)} ({msg})")
        self.code = code


class qvts_model_desc(C.Structure):
    _fields_ = [("height", C.c_int32), ("width", C.c_int32), ("occupancy", C.c_void_p), ("goal", C.c_int32),
                ("action_mask", C.c_uint32), ("p_intended", C.c_double), ("p_stay", C.c_double),
                ("p_lateral", C.c_double), ("sensor_acc", C.c_double), ("gamma", C.c_double),
                ("device", C.c_int32)]


class qvts_plan_cfg(C.Structure):
    _fields_ = [("depth", C.c_int32), ("n_samples", C.c_int32), ("seed", C.c_uint32), ("step", C.c_uint32),
                ("episode", C.c_uint32), ("want_trace", C.c_int32), ("leaf_bound", C.c_int32),
                ("sampler", C.c_int32)]


class qvts_plan_result(C.Structure):
    _fields_ = [("action", C.c_int32), ("n_actions", C.c_int32), ("q_root", C.c_double * 9),
                ("n_vnodes", C.c_int64 * 9), ("n_belief_updates", C.c_int64), ("device_ms", C.c_double),
                ("shard_level", C.c_int32), ("n_flag_candidates", C.c_int64), ("n_tiles_skipped", C.c_int64)]


class qvts_bf_cfg(C.Structure):
    _fields_ = [("n_samples", C.c_int32), ("seed", C.c_uint32), ("step", C.c_uint32), ("episode", C.c_uint32),
                ("sampler", C.c_int32), ("max_expansions", C.c_int32), ("max_depth", C.c_int32),
                ("gap_tol", C.c_double), ("time_budget_ms", C.c_double), ("reuse", C.c_int32)]


class qvts_bf_result(C.Structure):
    _fields_ = [("action", C.c_int32), ("n_actions", C.c_int32), ("n_expansions", C.c_int32),
                ("stop_reason", C.c_int32), ("n_vnodes", C.c_int64), ("U", C.c_double), ("L", C.c_double),
                ("u_q", C.c_double * 9), ("l_q", C.c_double * 9), ("device_ms", C.c_double)]


class qvts_profile(C.Structure):
    _fields_ = [("launches", C.c_int64 * 8), ("ms", C.c_double * 8), ("leaf_cells", C.c_int64),
                ("hist_cells", C.c_int64), ("correct_cells_written", C.c_int64), ("total_launches", C.c_int64)]


PROFILE_CLASSES = ["hist_leaf", "hist", "reduce_leaf", "reduce", "scan", "correct", "backup", "other"]


ALLREDUCE_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p)


class qvts_comm(C.Structure):
    _fields_ = [("rank", C.c_int32), ("nranks", C.c_int32), ("min_nodes_per_rank", C.c_int32),
                ("allreduce_sum_f64", ALLREDUCE_FN), ("ctx", C.c_void_p)]


class qvts_episode_cfg(C.Structure):
    _fields_ = [("n_episodes", C.c_int32), ("max_steps", C.c_int32), ("stop_patience", C.c_int32),
                ("planner", C.c_int32), ("depth", C.c_int32), ("n_samples", C.c_int32), ("seed", C.c_uint32),
                ("b0_dev", C.c_void_p), ("log_actions", C.c_void_p), ("log_obs", C.c_void_p),
                ("log_states", C.c_void_p)]


class qvts_episode_record(C.Structure):
    _fields_ = [("outcome", C.c_int32), ("steps", C.c_int32), ("collisions", C.c_int32), ("x0", C.c_int32),
                ("x_final", C.c_int32), ("disc_return", C.c_double)]


_lib = None


def lib() -> C.CDLL:
    """Load libqvts.so (built in-tree by __graft_entry__.build() / make -C csrc)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"libqvts.so not built at {LIB_PATH}: run `make -C {_HERE}/csrc` "
                              "(there is no CPU fallback)")
        L = C.CDLL(LIB_PATH)
        vp, st = C.c_void_p, C.c_int
        L.qvts_model_create.argtypes = [C.POINTER(qvts_model_desc), C.POINTER(vp)]
        L.qvts_model_destroy.argtypes = [vp]
        L.qvts_model_destroy.restype = None
        L.qvts_last_error.restype = C.c_char_p
        L.qvts_model_info.argtypes = [vp, C.POINTER(C.c_int32), vp, C.POINTER(C.c_int64)]
        L.qvts_model_tables.argtypes = [vp, vp, vp]
        L.qvts_value_iteration.argtypes = [vp, C.c_double, C.c_int32, C.POINTER(C.c_int32),
                                           C.POINTER(C.c_double), vp]
        L.qvts_get_q.argtypes = [vp, vp]
        L.qvts_fib_iteration.argtypes = [vp, C.c_double, C.c_int32, C.POINTER(C.c_int32), C.POINTER(C.c_double), vp]
        L.qvts_get_alpha.argtypes = [vp, vp]
        L.qvts_pbvi.argtypes = [vp, vp, C.c_int32, C.c_int32, C.c_uint32, C.c_int32, C.POINTER(C.c_int32), vp]
        L.qvts_get_pbvi.argtypes = [vp, vp, vp, vp, C.POINTER(C.c_int32)]
        L.qvts_plan_best_first.argtypes = [vp, vp, C.POINTER(qvts_bf_cfg), C.POINTER(qvts_bf_result), vp]
        L.qvts_trace_best_first.argtypes = [vp, C.POINTER(C.c_int64), C.POINTER(C.c_int32)] + [vp] * 10
        L.qvts_bf_advance.argtypes = [vp, C.c_int32, C.c_int32, C.POINTER(C.c_int32), vp]
        L.qvts_belief_update.argtypes = [vp, vp, C.c_int32, C.c_int32, vp, C.POINTER(C.c_double), vp]
        L.qvts_belief_update_batch.argtypes = [vp, vp, C.c_int64, C.c_int32, vp, vp, vp, C.c_int64, vp, vp]
        L.qvts_plan_step.argtypes = [vp, vp, C.POINTER(qvts_plan_cfg), C.POINTER(qvts_comm),
                                     C.POINTER(qvts_plan_result), vp]
        L.qvts_trace_qnodes.argtypes = [vp, C.c_int32, vp, vp, vp, vp, vp, vp]
        L.qvts_trace_vnodes.argtypes = [vp, C.c_int32, vp, vp, vp, vp, vp]
        L.qvts_trace_leaf_values.argtypes = [vp, vp]
        L.qvts_trace_belief.argtypes = [vp, C.c_int32, C.c_int64, vp]
        L.qvts_trace_state_draws.argtypes = [vp, C.c_int32, vp]
        L.qvts_trace_counts.argtypes = [vp, C.POINTER(C.c_int32), vp, vp]
        L.qvts_set_profiling.argtypes = [vp, C.c_int32]
        L.qvts_get_profile.argtypes = [vp, C.POINTER(qvts_profile)]
        L.qvts_run_episodes.argtypes = [vp, C.POINTER(qvts_episode_cfg), C.POINTER(qvts_comm),
                                        vp, vp]
        for f in EXPORTS:
            if f not in ("qvts_model_destroy", "qvts_last_error"):
                getattr(L, f).restype = st
        _lib = L
    return _lib


def qvts_last_error() -> str:
    return lib().qvts_last_error().decode()


def _check(code: int, where: str):
    if code != QVTS_OK:
        raise QvtsError(code, where, qvts_last_error())


def _ptr(a) -> int:
    """Raw pointer of a torch tensor or numpy array (marshalling only)."""
    if a is None:
        return 0
    if isinstance(a, np.ndarray):
        return a.ctypes.data
    return a.data_ptr()


def _stream(stream) -> int:
    if stream is not None:
        return int(stream)
    import torch
    return torch.cuda.current_stream().cuda_stream


# ---- ABI wrappers (same names as the C entry points) -----------------------------------------
def qvts_model_create(height, width, occupancy, goal, action_mask=0x1FF, p_intended=0.8, p_stay=0.1,
                      p_lateral=0.05, sensor_acc=0.95, gamma=0.95, device=0):
    occ = np.ascontiguousarray(occupancy, dtype=np.uint8)
    d = qvts_model_desc(int(height), int(width), occ.ctypes.data, int(goal), int(action_mask), p_intended,
                        p_stay, p_lateral, sensor_acc, gamma, int(device))
    h = C.c_void_p()
    _check(lib().qvts_model_create(C.byref(d), C.byref(h)), "qvts_model_create")
    return h.value


def qvts_model_destroy(h):
    lib().qvts_model_destroy(h)


def qvts_model_info(h):
    na = C.c_int32()
    ids = (C.c_int32 * 9)()
    nc = C.c_int64()
    _check(lib().qvts_model_info(h, C.byref(na), ids, C.byref(nc)), "qvts_model_info")
    return na.value, list(ids)[:na.value], nc.value


def qvts_model_tables(h, n_actions, n_cells):
    R = np.zeros((n_actions, n_cells), np.float32)
    sig = np.zeros(n_cells, np.uint8)
    _check(lib().qvts_model_tables(h, R.ctypes.data, sig.ctypes.data), "qvts_model_tables")
    return R, sig


def qvts_value_iteration(h, eps=1e-9, max_sweeps=100000, stream=None):
    sw, res = C.c_int32(), C.c_double()
    code = lib().qvts_value_iteration(h, eps, max_sweeps, C.byref(sw), C.byref(res), _stream(stream))
    if code not in (QVTS_OK, 4):
        _check(code, "qvts_value_iteration")
    return code, sw.value, res.value


def qvts_get_q(h, n_actions, n_cells):
    q = np.zeros((n_actions, n_cells), np.float64)
    _check(lib().qvts_get_q(h, q.ctypes.data), "qvts_get_q")
    return q


def qvts_fib_iteration(h, eps=1e-9, max_sweeps=100000, stream=None):
    sw, res = C.c_int32(), C.c_double()
    code = lib().qvts_fib_iteration(h, eps, max_sweeps, C.byref(sw), C.byref(res), _stream(stream))
    if code not in (QVTS_OK, 4):
        _check(code, "qvts_fib_iteration")
    return code, sw.value, res.value


def qvts_get_alpha(h, n_actions, n_cells):
    a = np.zeros((n_actions, n_cells), np.float64)
    _check(lib().qvts_get_alpha(h, a.ctypes.data), "qvts_get_alpha")
    return a


def qvts_belief_update_batch(h, b_dev, actions, zs, out_dev, stream=None):
    """Batched Eq. 3: b_dev / out_dev are [n][>= H*W] fp32 device tensors; returns P(z|b,a) [n]."""
    acts = np.ascontiguousarray(actions, dtype=np.int32)
    z = np.ascontiguousarray(zs, dtype=np.int32)
    n = len(acts)
    p = np.zeros(max(1, n))
    _check(lib().qvts_belief_update_batch(h, _ptr(b_dev), int(b_dev.stride(0)) if n else 0, n, acts.ctypes.data,
                                          z.ctypes.data, _ptr(out_dev), int(out_dev.stride(0)) if n else 0,
                                          p.ctypes.data, _stream(stream)), "qvts_belief_update_batch")
    return p[:n]


def qvts_pbvi(h, b0_dev=None, expansions=3, max_points=16, seed=1, sweeps=30, stream=None):
    n = C.c_int32()
    _check(lib().qvts_pbvi(h, _ptr(b0_dev) if b0_dev is not None else None, int(expansions), int(max_points),
                           int(seed), int(sweeps), C.byref(n), _stream(stream)), "qvts_pbvi")
    return n.value


def qvts_get_pbvi(h, n_points, n_cells):
    """-> (points [n_points][n_cells] fp64, alphas [n_alpha][n_cells] fp64, actions [n_points])."""
    nal = C.c_int32()
    _check(lib().qvts_get_pbvi(h, None, None, None, C.byref(nal)), "qvts_get_pbvi")
    pts = np.zeros((n_points, n_cells), np.float64)
    al = np.zeros((nal.value, n_cells), np.float64)
    act = np.zeros(n_points, np.int32)
    _check(lib().qvts_get_pbvi(h, pts.ctypes.data, al.ctypes.data, act.ctypes.data, None), "qvts_get_pbvi")
    return pts, al, act


def qvts_plan_best_first(h, root_dev, n_samples, max_expansions, max_depth=8, gap_tol=0.0, seed=1, step=0,
                         episode=0, sampler=QVTS_SAMPLER_MARGINAL, time_budget_ms=0.0, reuse=False, stream=None):
    cfg = qvts_bf_cfg(n_samples, seed, step, episode, sampler, max_expansions, max_depth, gap_tol, time_budget_ms,
                      1 if reuse else 0)
    res = qvts_bf_result()
    _check(lib().qvts_plan_best_first(h, _ptr(root_dev), C.byref(cfg), C.byref(res), _stream(stream)),
           "qvts_plan_best_first")
    return res


def qvts_bf_advance(h, action, z, stream=None):
    """Re-root the last best-first tree at its (action, z) child; True when the subtree is kept."""
    r = C.c_int32()
    _check(lib().qvts_bf_advance(h, int(action), int(z), C.byref(r), _stream(stream)), "qvts_bf_advance")
    return bool(r.value)


def qvts_trace_best_first(h):
    """-> dict: per V-node arrays path/depth/f/U/L/H/E/expanded, exp_order, root_trace [(U, L)]."""
    nv, ne = C.c_int64(), C.c_int32()
    _check(lib().qvts_trace_best_first(h, C.byref(nv), C.byref(ne), *([None] * 10)), "qvts_trace_best_first")
    n, k = nv.value, ne.value
    out = dict(path=np.zeros(n, np.uint64), depth=np.zeros(n, np.int32), f=np.zeros(n, np.int32),
               U=np.zeros(n), L=np.zeros(n), H=np.zeros(n), E=np.zeros(n, np.int32),
               expanded=np.zeros(n, np.int32), exp_order=np.zeros(k, np.int32), root_trace=np.zeros((k + 1, 2)))
    order = ("path", "depth", "f", "U", "L", "H", "E", "expanded", "exp_order", "root_trace")
    _check(lib().qvts_trace_best_first(h, None, None, *[out[o].ctypes.data for o in order]), "qvts_trace_best_first")
    return out


def qvts_belief_update(h, b_dev, action, z, out_dev, stream=None):
    p = C.c_double()
    _check(lib().qvts_belief_update(h, _ptr(b_dev), int(action), int(z), _ptr(out_dev), C.byref(p),
                                    _stream(stream)), "qvts_belief_update")
    return p.value


def qvts_plan_step(h, root_dev, depth, n_samples, seed=1, step=0, episode=0, want_trace=False, comm=None,
                   stream=None, leaf_bound=QVTS_LEAF_QMDP, sampler=QVTS_SAMPLER_MARGINAL) -> qvts_plan_result:
    cfg = qvts_plan_cfg(int(depth), int(n_samples), int(seed), int(step), int(episode), 1 if want_trace else 0,
                        int(leaf_bound), int(sampler))
    res = qvts_plan_result()
    _check(lib().qvts_plan_step(h, _ptr(root_dev), C.byref(cfg), C.byref(comm) if comm is not None else None,
                                C.byref(res), _stream(stream)), "qvts_plan_step")
    return res


def qvts_trace_counts(h):
    depth = C.c_int32()
    nv = (C.c_int64 * 10)()
    nq = (C.c_int64 * 10)()
    _check(lib().qvts_trace_counts(h, C.byref(depth), nv, nq), "qvts_trace_counts")
    D = depth.value
    return D, list(nv)[:D], list(nq)[:D]


def qvts_trace_qnodes(h, level, n_q, n_samples=0, with_draws=False):
    path = np.zeros(n_q, np.uint64); R = np.zeros(n_q); P = np.zeros((n_q, 16)); cnt = np.zeros((n_q, 16), np.uint16)
    Q = np.zeros(n_q); z = np.zeros((n_q, max(1, n_samples)), np.uint8) if with_draws else None
    _check(lib().qvts_trace_qnodes(h, level, path.ctypes.data, R.ctypes.data, P.ctypes.data, cnt.ctypes.data,
                                   Q.ctypes.data, z.ctypes.data if with_draws else None), "qvts_trace_qnodes")
    return dict(path=path, R=R, P=P, cnt=cnt, Q=Q, z=z)


def qvts_trace_vnodes(h, level, n_v):
    path = np.zeros(n_v, np.uint64); parent = np.zeros(n_v, np.int32); z = np.zeros(n_v, np.int32)
    f = np.zeros(n_v, np.int32); V = np.zeros(n_v)
    _check(lib().qvts_trace_vnodes(h, level, path.ctypes.data, parent.ctypes.data, z.ctypes.data, f.ctypes.data,
                                   V.ctypes.data), "qvts_trace_vnodes")
    return dict(path=path, parent_q=parent, z=z, f=f, V=V)


def qvts_trace_leaf_values(h, n_q):
    V = np.zeros((n_q, 16))
    _check(lib().qvts_trace_leaf_values(h, V.ctypes.data), "qvts_trace_leaf_values")
    return V


def qvts_trace_state_draws(h, level, n_q, n_samples):
    x = np.zeros((n_q, max(1, n_samples)), np.int32)
    _check(lib().qvts_trace_state_draws(h, level, x.ctypes.data), "qvts_trace_state_draws")
    return x


def qvts_trace_belief(h, level, index, n_cells):
    out = np.zeros(n_cells, np.float32)
    _check(lib().qvts_trace_belief(h, level, index, out.ctypes.data), "qvts_trace_belief")
    return out


def qvts_set_profiling(h, enable=True):
    _check(lib().qvts_set_profiling(h, 1 if enable else 0), "qvts_set_profiling")


def qvts_get_profile(h) -> dict:
    p = qvts_profile()
    _check(lib().qvts_get_profile(h, C.byref(p)), "qvts_get_profile")
    return dict(launches=dict(zip(PROFILE_CLASSES, list(p.launches))), ms=dict(zip(PROFILE_CLASSES, list(p.ms))),
                leaf_cells=p.leaf_cells, hist_cells=p.hist_cells, correct_cells_written=p.correct_cells_written,
                total_launches=p.total_launches)


def qvts_run_episodes(h, n_episodes, max_steps=500, stop_patience=3, planner=QVTS_PLANNER_QVTS, depth=3,
                      n_samples=8, seed=1, b0_dev=None, comm=None, stream=None, logs=False):
    """Returns (records as a dict of numpy arrays, logs dict or None)."""
    la = lz = lx = None
    if logs:
        la = np.full((n_episodes, max_steps), -1, np.int32)
        lz = np.full((n_episodes, max_steps), -1, np.int32)
        lx = np.full((n_episodes, max_steps), -1, np.int32)
    cfg = qvts_episode_cfg(int(n_episodes), int(max_steps), int(stop_patience), int(planner), int(depth),
                           int(n_samples), int(seed), _ptr(b0_dev) or None, _ptr(la) or None, _ptr(lz) or None,
                           _ptr(lx) or None)
    recs = (qvts_episode_record * max(1, n_episodes))()
    _check(lib().qvts_run_episodes(h, C.byref(cfg), C.byref(comm) if comm is not None else None, recs,
                                   _stream(stream)), "qvts_run_episodes")
    out = {k: np.array([getattr(recs[i], k) for i in range(n_episodes)])
           for k in ("outcome", "steps", "collisions", "x0", "x_final", "disc_return")}
    return out, (dict(actions=la, obs=lz, states=lx) if logs else None)


# ---- multi-rank plumbing: the all-reduce callback runs torch.distributed (NCCL) ----------------
class _CudaArray:
    def __init__(self, ptr, n):
        self.__cuda_array_interface__ = {"shape": (int(n),), "typestr": "<f8", "data": (int(ptr), False),
                                         "version": 2, "strides": None, "stream": None}


def make_torch_comm(min_nodes_per_rank=16):
    """qvts_comm whose all-reduce is torch.distributed.all_reduce(SUM) on the library's stream."""
    import torch
    import torch.distributed as dist

    def _allreduce(ctx, buf, count, stream):
        try:
            s = torch.cuda.ExternalStream(int(stream)) if stream else torch.cuda.current_stream()
            with torch.cuda.stream(s):
                t = torch.as_tensor(_CudaArray(buf, count), device="cuda")
                if dist.get_backend() == "nccl":
                    dist.all_reduce(t, op=dist.ReduceOp.SUM)
                else:                                   # host backends (gloo): stage through host
                    h = t.cpu()
                    dist.all_reduce(h, op=dist.ReduceOp.SUM)
                    t.copy_(h)
            return 0
        except Exception:  # noqa: BLE001 - surfaced as QVTS_ERR_COMM
            return 1

    cb = ALLREDUCE_FN(_allreduce)
    comm = qvts_comm(dist.get_rank(), dist.get_world_size(), int(min_nodes_per_rank), cb, None)
    comm._keep = cb  # keep the callback alive
    return comm


def make_callback_comm(rank, nranks, fn, min_nodes_per_rank=16):
    """qvts_comm around an arbitrary Python callable fn(ptr, count, stream) -> None (tests)."""
    def _cb(ctx, buf, count, stream):
        try:
            fn(buf, count, stream)
            return 0
        except Exception:  # noqa: BLE001
            return 1
    cb = ALLREDUCE_FN(_cb)
    comm = qvts_comm(int(rank), int(nranks), int(min_nodes_per_rank), cb, None)
    comm._keep = cb
    return comm


class Model:
    """Holds a qvts_model handle; methods forward to the ABI wrappers above."""

    def __init__(self, gmap, action_mask=0x1FF, p_intended=0.8, p_stay=0.1, p_lateral=0.05, sensor_acc=0.95,
                 gamma=0.95, device=0):
        self.h = qvts_model_create(gmap.height, gmap.width, gmap.occupancy, gmap.goal, action_mask, p_intended,
                                   p_stay, p_lateral, sensor_acc, gamma, device)
        self.n_actions, self.action_ids, self.n_cells = qvts_model_info(self.h)
        self.gmap = gmap

    def close(self):
        if getattr(self, "h", None):
            qvts_model_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:  # noqa: BLE001
            pass

    def value_iteration(self, eps=1e-9, max_sweeps=100000):
        return qvts_value_iteration(self.h, eps, max_sweeps)

    def q(self):
        return qvts_get_q(self.h, self.n_actions, self.n_cells)

    def fib_iteration(self, eps=1e-9, max_sweeps=100000):
        return qvts_fib_iteration(self.h, eps, max_sweeps)

    def alpha(self):
        return qvts_get_alpha(self.h, self.n_actions, self.n_cells)

    def pbvi(self, b0_dev=None, expansions=3, max_points=16, seed=1, sweeps=30):
        """PBVI lower bound on the GPU -> (points, alphas, actions) as host fp64 / int32 arrays."""
        n = qvts_pbvi(self.h, b0_dev, expansions, max_points, seed, sweeps)
        return qvts_get_pbvi(self.h, n, self.n_cells)

    def tables(self):
        return qvts_model_tables(self.h, self.n_actions, self.n_cells)

    def belief_update_batch(self, b_dev, actions, zs, out_dev):
        return qvts_belief_update_batch(self.h, b_dev, actions, zs, out_dev)

    def belief_update(self, b_dev, action, z, out_dev):
        return qvts_belief_update(self.h, b_dev, action, z, out_dev)

    def plan_step(self, root_dev, depth, n_samples, **kw):
        return qvts_plan_step(self.h, root_dev, depth, n_samples, **kw)

    def plan_best_first(self, root_dev, n_samples, max_expansions, **kw):
        """Anytime best-first QVTS (needs fib_iteration and pbvi first)."""
        return qvts_plan_best_first(self.h, root_dev, n_samples, max_expansions, **kw)

    def trace_best_first(self):
        return qvts_trace_best_first(self.h)

    def bf_advance(self, action, z):
        return qvts_bf_advance(self.h, action, z)

    def run_episodes(self, n_episodes, **kw):
        return qvts_run_episodes(self.h, n_episodes, **kw)

    def trace(self, with_draws=False, n_samples=0, beliefs=False, with_states=False):
        """Pull the whole tree of the last plan step to the host (small configs).  with_draws and
        the leaf values need a plan step run with want_trace=True; with_states (the ancestral
        sampler's state index per draw) also needs sampler=QVTS_SAMPLER_ANCESTRAL."""
        D, nv, nq = qvts_trace_counts(self.h)
        levels = []
        for d in range(D):
            q = qvts_trace_qnodes(self.h, d, nq[d] * self.n_actions, n_samples, with_draws)
            if with_states:
                q["x"] = qvts_trace_state_draws(self.h, d, nq[d] * self.n_actions, n_samples)
            v = qvts_trace_vnodes(self.h, d, nv[d])
            if beliefs and d > 0:
                v["belief"] = np.stack([qvts_trace_belief(self.h, d, i, self.n_cells) for i in range(nv[d])]) \
                    if nv[d] else np.zeros((0, self.n_cells), np.float32)
            levels.append(dict(q=q, v=v))
        leaf = qvts_trace_leaf_values(self.h, nq[D - 1] * self.n_actions) if with_draws else None
        return dict(depth=D, levels=levels, leafV=leaf)
