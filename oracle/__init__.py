"""TEST INFRASTRUCTURE ONLY — ctypes wrapper around the fp64 C oracle (qvts_oracle.c).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs may
import this package.  It never imports the CUDA library package and vice versa.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# QVTS_ORACLE_LIB: load a prebuilt oracle library instead (tests/oracle_mutations.py runs the pins
# against deliberately broken copies to show they catch plausible mistakes)
_LIB_PATH = os.environ.get("QVTS_ORACLE_LIB") or os.path.join(_HERE, "liboracle.so")

OK, ERR_INVALID_ARG, ERR_INVALID_MODEL, ERR_NOT_CONVERGED, ERR_ZERO_LIKELIHOOD = 0, 1, 2, 4, 5
MODE_FREQ, MODE_EXACT, MODE_BRUTE = 0, 1, 2
PLANNER_QVTS, PLANNER_MDP, PLANNER_ASTAR = 0, 1, 2
SAMPLER_MARGINAL, SAMPLER_ANCESTRAL = 0, 1


def build() -> str:
    if os.environ.get("QVTS_ORACLE_LIB"):
        return _LIB_PATH
    src = os.path.join(_HERE, "qvts_oracle.c")
    if not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(src):
        subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = C.CDLL(build())
        _declare(_lib)
    return _lib


_dp = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")
_u8p = np.ctypeslib.ndpointer(dtype=np.uint8, flags="C_CONTIGUOUS")
_u16p = np.ctypeslib.ndpointer(dtype=np.uint16, flags="C_CONTIGUOUS")
_i32p = np.ctypeslib.ndpointer(dtype=np.int32, flags="C_CONTIGUOUS")
_i64p = np.ctypeslib.ndpointer(dtype=np.int64, flags="C_CONTIGUOUS")
_u64p = np.ctypeslib.ndpointer(dtype=np.uint64, flags="C_CONTIGUOUS")
_u32p = np.ctypeslib.ndpointer(dtype=np.uint32, flags="C_CONTIGUOUS")


class PlanCfg(C.Structure):
    _fields_ = [("depth", C.c_int), ("n_samples", C.c_int), ("mode", C.c_int), ("threads", C.c_int),
                ("seed", C.c_uint32), ("step", C.c_uint32), ("episode", C.c_uint32),
                ("sampler", C.c_int), ("n_replay", C.c_int), ("replay_path", C.c_void_p),
                ("replay_j", C.c_void_p), ("replay_z", C.c_void_p), ("replay_x", C.c_void_p)]


class BfCfg(C.Structure):
    _fields_ = [("expansions", C.c_int), ("max_depth", C.c_int), ("gap_tol", C.c_double),
                ("n_replay", C.c_int), ("replay_path", C.c_void_p), ("replay_tol", C.c_double)]


class EpisodeCfg(C.Structure):
    _fields_ = [("planner", C.c_int), ("depth", C.c_int), ("n_samples", C.c_int),
                ("max_steps", C.c_int), ("stop_patience", C.c_int),
                ("seed", C.c_uint32), ("episode", C.c_uint32)]


class EpisodeRecord(C.Structure):
    _fields_ = [("outcome", C.c_int32), ("steps", C.c_int32), ("collisions", C.c_int32),
                ("x0", C.c_int32), ("x_final", C.c_int32), ("disc_return", C.c_double)]


class BfTree:
    """A persistent oracle best-first tree: plan, then advance(a, z) + cont(...) for tree reuse."""

    def __init__(self, model, alphaU, alphaL, actL, b0, n, expansions, max_depth=8, gap_tol=0.0, seed=1, step=0,
                 episode=0, mode=0, sampler=0, replay=None, replay_tol=1e-4):
        self.m = model
        self.aU = np.ascontiguousarray(alphaU, dtype=np.float64)
        self.aL = np.ascontiguousarray(alphaL, dtype=np.float64)
        self.acts = np.ascontiguousarray(actL, dtype=np.int32)
        cfg, bc, _keep = self._cfgs(n, expansions, max_depth, gap_tol, seed, step, episode, mode, sampler, replay,
                                    replay_tol)
        self.h = lib().or_bf_plan(model._h, self.aU, self.aU.shape[0], self.aL, self.aL.shape[0], self.acts,
                                  np.ascontiguousarray(b0, dtype=np.float64), C.byref(cfg), C.byref(bc))
        if not self.h:
            raise ValueError("or_bf_plan rejected its arguments")

    def _cfgs(self, n, expansions, max_depth, gap_tol, seed, step, episode, mode, sampler, replay, replay_tol):
        cfg, k = self.m._cfg(0, n, seed, step, episode, mode, 0, None, sampler)
        rp = np.ascontiguousarray(replay if replay is not None else [], dtype=np.uint64)
        bc = BfCfg(expansions, max_depth, gap_tol, len(rp), rp.ctypes.data if len(rp) else None, replay_tol)
        return cfg, bc, (k, rp)

    def cont(self, n, expansions, max_depth=8, gap_tol=0.0, seed=1, step=0, episode=0, mode=0, sampler=0,
             replay=None, replay_tol=1e-4):
        cfg, bc, _keep = self._cfgs(n, expansions, max_depth, gap_tol, seed, step, episode, mode, sampler, replay,
                                    replay_tol)
        st = lib().or_bf_continue(self.h, self.aU, self.aU.shape[0], self.aL, self.aL.shape[0], self.acts,
                                  C.byref(cfg), C.byref(bc))
        if st != OK:
            raise OracleError(st, "or_bf_continue")
        return self.result()

    def advance(self, a_id, z):
        return bool(lib().or_bf_advance(self.h, int(a_id), int(z)))

    def belief(self, i):
        out = np.zeros(self.m.nx)
        lib().or_bf_belief(self.h, int(i), out)
        return out

    def result(self):
        L_, h = lib(), self.h
        out = {}
        vals = [C.c_int() for _ in range(6)]
        L_.or_bf_summary(h, *[C.byref(v) for v in vals])
        for k, v in zip(("action", "stop", "n_exp", "n_v", "subs", "mism"), vals):
            out[k] = v.value
        U, Lo = C.c_double(), C.c_double()
        UQ, LQ = np.zeros(self.m.na), np.zeros(self.m.na)
        L_.or_bf_root(h, C.byref(U), C.byref(Lo), UQ, LQ)
        out.update(U=U.value, L=Lo.value, UQ=UQ, LQ=LQ, root=L_.or_bf_root_index(h))
        out["expanded"] = np.array([L_.or_bf_expanded(h, k) for k in range(out["n_exp"])], dtype=np.uint64)
        rt = []
        for k in range(out["n_exp"] + 1):
            L_.or_bf_root_trace(h, k, C.byref(U), C.byref(Lo))
            rt.append((U.value, Lo.value))
        out["root_trace"] = np.array(rt)
        cols = {k: [] for k in ("path", "depth", "f", "w", "U", "L", "H", "E", "expanded")}
        p, d, f, E, ex = C.c_uint64(), C.c_int(), C.c_int(), C.c_int(), C.c_int()
        w, u, l, hh = C.c_double(), C.c_double(), C.c_double(), C.c_double()
        for i in range(out["n_v"]):
            L_.or_bf_vnode(h, i, C.byref(p), C.byref(d), C.byref(f), C.byref(w), C.byref(u), C.byref(l),
                           C.byref(hh), C.byref(E), C.byref(ex))
            for k, v in zip(cols, (p, d, f, w, u, l, hh, E, ex)):
                cols[k].append(v.value)
        out["v"] = {k: np.array(v, dtype=np.uint64 if k == "path" else None) for k, v in cols.items()}
        return out

    def close(self):
        if getattr(self, "h", None):
            lib().or_bf_free(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:  # noqa: BLE001
            pass


def bf_q_update(R, gamma, w, U, L, H, E):
    """Alg. 6 on explicit child values -> (U_Q, L_Q, H_Q, E_Q)."""
    out = [C.c_double(), C.c_double(), C.c_double(), C.c_int()]
    lib().or_bf_q_update(R, gamma, len(w), *[np.ascontiguousarray(a, dtype=np.float64) for a in (w, U, L, H)],
                         np.ascontiguousarray(E, dtype=np.int32), *[C.byref(o) for o in out])
    return tuple(o.value for o in out)


def bf_v_update(UQ, LQ, HQ, EQ):
    """Alg. 7 (argmax-U_Q child) on explicit Q values -> (U, L, H, E)."""
    out = [C.c_double(), C.c_double(), C.c_double(), C.c_int()]
    lib().or_bf_v_update(len(UQ), *[np.ascontiguousarray(a, dtype=np.float64) for a in (UQ, LQ, HQ)],
                         np.ascontiguousarray(EQ, dtype=np.int32), *[C.byref(o) for o in out])
    return tuple(o.value for o in out)


def _declare(L):
    vp = C.c_void_p
    L.or_grid_model_create.restype = vp
    L.or_grid_model_create.argtypes = [C.c_int, C.c_int, _u8p, C.c_int, C.c_uint, C.c_double, C.c_double,
                                       C.c_double, C.c_double, C.c_double, C.POINTER(C.c_int)]
    L.or_dense_model_create.restype = vp
    L.or_dense_model_create.argtypes = [C.c_int, C.c_int, C.c_int, _dp, _dp, _dp, C.c_double,
                                        C.POINTER(C.c_int)]
    L.or_model_free.argtypes = [vp]
    for f in ("or_num_states", "or_num_actions", "or_num_obs"):
        getattr(L, f).argtypes = [vp]
    L.or_action_id.argtypes = [vp, C.c_int]
    L.or_T.restype = C.c_double
    L.or_T.argtypes = [vp, C.c_int, C.c_int, C.c_int]
    L.or_Tprime.restype = C.c_double
    L.or_Tprime.argtypes = [vp, C.c_int, C.c_int, C.c_int]
    L.or_O.restype = C.c_double
    L.or_O.argtypes = [vp, C.c_int, C.c_int]
    L.or_R.restype = C.c_double
    L.or_R.argtypes = [vp, C.c_int, C.c_int]
    L.or_sig.argtypes = [vp, C.c_int]
    L.or_occ.argtypes = [vp, C.c_int]
    L.or_philox4x32_10.argtypes = [_u32p, _u32p, _u32p]
    L.or_uniform.restype = C.c_double
    L.or_uniform.argtypes = [C.c_uint32]
    L.or_inverse_cdf.argtypes = [_dp, C.c_int, C.c_double, C.POINTER(C.c_int)]
    L.or_predict.argtypes = [vp, _dp, C.c_int, _dp]
    L.or_marginal.argtypes = [vp, _dp, _dp]
    L.or_belief_reward.restype = C.c_double
    L.or_belief_reward.argtypes = [vp, _dp, C.c_int]
    L.or_belief_update.argtypes = [vp, _dp, C.c_int, C.c_int, _dp, C.POINTER(C.c_double)]
    L.or_value_iteration.argtypes = [vp, C.c_double, C.c_int, _dp, _dp, C.POINTER(C.c_int),
                                     C.POINTER(C.c_double)]
    L.or_fib.argtypes = [vp, C.c_double, C.c_int, _dp, C.POINTER(C.c_int), C.POINTER(C.c_double)]
    L.or_pbvi_build.restype = vp
    L.or_pbvi_build.argtypes = [vp, _dp, C.c_int, C.c_int, C.c_uint32, C.c_int]
    L.or_pbvi_free.argtypes = [vp]
    L.or_pbvi_npoints.argtypes = [vp]
    L.or_pbvi_nalpha.argtypes = [vp]
    L.or_pbvi_point.argtypes = [vp, C.c_int, _dp]
    L.or_pbvi_alpha.argtypes = [vp, C.c_int, _dp, C.POINTER(C.c_int)]
    L.or_pbvi_value.restype = C.c_double
    L.or_pbvi_value.argtypes = [vp, _dp]
    L.or_bf_q_update.argtypes = [C.c_double, C.c_double, C.c_int, _dp, _dp, _dp, _dp, _i32p,
                                 C.POINTER(C.c_double), C.POINTER(C.c_double), C.POINTER(C.c_double),
                                 C.POINTER(C.c_int)]
    L.or_bf_v_update.argtypes = [C.c_int, _dp, _dp, _dp, _i32p, C.POINTER(C.c_double), C.POINTER(C.c_double),
                                 C.POINTER(C.c_double), C.POINTER(C.c_int)]
    L.or_bf_plan.restype = vp
    L.or_bf_plan.argtypes = [vp, _dp, C.c_int, _dp, C.c_int, _i32p, _dp, C.POINTER(PlanCfg), C.POINTER(BfCfg)]
    L.or_bf_free.argtypes = [vp]
    L.or_bf_continue.argtypes = [vp, _dp, C.c_int, _dp, C.c_int, _i32p, C.POINTER(PlanCfg), C.POINTER(BfCfg)]
    L.or_bf_advance.argtypes = [vp, C.c_int, C.c_int]
    L.or_bf_root_index.argtypes = [vp]
    L.or_bf_belief.argtypes = [vp, C.c_int, _dp]
    L.or_bf_summary.argtypes = [vp] + [C.POINTER(C.c_int)] * 6
    L.or_bf_root.argtypes = [vp, C.POINTER(C.c_double), C.POINTER(C.c_double), _dp, _dp]
    L.or_bf_vnode.argtypes = [vp, C.c_int, C.POINTER(C.c_uint64), C.POINTER(C.c_int), C.POINTER(C.c_int),
                              C.POINTER(C.c_double), C.POINTER(C.c_double), C.POINTER(C.c_double),
                              C.POINTER(C.c_double), C.POINTER(C.c_int), C.POINTER(C.c_int)]
    L.or_bf_expanded.restype = C.c_uint64
    L.or_bf_expanded.argtypes = [vp, C.c_int]
    L.or_bf_root_trace.argtypes = [vp, C.c_int, C.POINTER(C.c_double), C.POINTER(C.c_double)]
    L.or_qmdp_value.restype = C.c_double
    L.or_qmdp_value.argtypes = [vp, _dp, _dp, C.POINTER(C.c_int)]
    L.or_trace_new.restype = vp
    L.or_trace_new.argtypes = [C.c_int]
    L.or_trace_free.argtypes = [vp]
    L.or_trace_nq.restype = C.c_int64
    L.or_trace_nq.argtypes = [vp]
    L.or_trace_nv.restype = C.c_int64
    L.or_trace_nv.argtypes = [vp]
    L.or_trace_nsamples.argtypes = [vp]
    L.or_trace_export_q.argtypes = [vp, _u64p, _i32p, _i32p, _dp, _dp, _u16p, _dp, _u8p, _u8p]
    L.or_trace_export_v.argtypes = [vp, _u64p, _i32p, _dp, _i32p, _i32p, _i64p]
    L.or_trace_belief.argtypes = [vp, C.c_int64, _dp]
    L.or_plan.argtypes = [vp, _dp, _dp, C.POINTER(PlanCfg), C.POINTER(C.c_int), _dp, vp]
    L.or_qnode_sample.argtypes = [vp, _dp, C.c_int, C.c_uint64, C.POINTER(PlanCfg), _dp,
                                  C.POINTER(C.c_double), _u8p, _u8p, _u16p]
    L.or_vnode_value.restype = C.c_double
    L.or_vnode_value.argtypes = [vp, _dp, _dp, C.c_uint64, C.c_int, C.POINTER(PlanCfg), _dp]
    L.or_run_episode.argtypes = [vp, _dp, _dp, C.POINTER(EpisodeCfg), C.POINTER(EpisodeRecord),
                                 _i32p, _i32p, _i32p]
    L.or_astar_action.argtypes = [vp, C.c_int]
    L.or_astar_length.argtypes = [vp, C.c_int]
    L.or_belief_mode.argtypes = [vp, _dp]
    L.or_ancestral_sample.argtypes = [vp, _dp, C.c_int, _u32p, _u32p]


class OracleError(RuntimeError):
    def __init__(self, code, what):
        super().__init__(f"{what}: oracle status {code}")
        self.code = code


def philox(ctr, key) -> np.ndarray:
    out = np.zeros(4, dtype=np.uint32)
    lib().or_philox4x32_10(np.asarray(ctr, dtype=np.uint32), np.asarray(key, dtype=np.uint32), out)
    return out


def uniform(w: int) -> float:
    return lib().or_uniform(int(w))


def inverse_cdf(p, u):
    flag = C.c_int(0)
    k = lib().or_inverse_cdf(np.ascontiguousarray(p, dtype=np.float64), len(p), float(u), C.byref(flag))
    return k, bool(flag.value)


@dataclass
class PlanResult:
    action: int
    qroot: np.ndarray
    trace: "Trace | None"


@dataclass
class Trace:
    q_path: np.ndarray
    q_level: np.ndarray
    q_action: np.ndarray
    q_R: np.ndarray
    q_P: np.ndarray
    q_cnt: np.ndarray
    q_Q: np.ndarray
    q_z: np.ndarray
    q_flag: np.ndarray
    v_path: np.ndarray
    v_level: np.ndarray
    v_V: np.ndarray
    v_z: np.ndarray
    v_f: np.ndarray
    v_belief: dict  # path -> np.ndarray (captured non-leaf beliefs)


class Model:
    """Oracle POMDP model: grid compile or a generic dense model."""

    def __init__(self, handle):
        self._h = handle
        L = lib()
        self.nx = L.or_num_states(handle)
        self.na = L.or_num_actions(handle)
        self.nz = L.or_num_obs(handle)
        self.action_ids = [L.or_action_id(handle, a) for a in range(self.na)]

    @classmethod
    def grid(cls, gmap, action_mask=0x1FF, p_int=0.8, p_stay=0.1, p_lat=0.05, acc=0.95, gamma=0.95):
        st = C.c_int(0)
        occ = np.ascontiguousarray(gmap.occupancy, dtype=np.uint8)
        h = lib().or_grid_model_create(gmap.height, gmap.width, occ, int(gmap.goal), int(action_mask),
                                       p_int, p_stay, p_lat, acc, gamma, C.byref(st))
        if not h:
            raise OracleError(st.value, "grid model")
        m = cls(h)
        m.gmap = gmap
        m.gamma = gamma
        return m

    @classmethod
    def dense(cls, T, O, R, gamma):
        T = np.ascontiguousarray(T, dtype=np.float64)
        nx, na, _ = T.shape
        nz = O.shape[1]
        st = C.c_int(0)
        h = lib().or_dense_model_create(nx, na, nz, T.reshape(-1),
                                        np.ascontiguousarray(O, dtype=np.float64).reshape(-1),
                                        np.ascontiguousarray(R, dtype=np.float64).reshape(-1),
                                        gamma, C.byref(st))
        if not h:
            raise OracleError(st.value, "dense model")
        m = cls(h)
        m.gamma = gamma
        return m

    def __del__(self):
        if getattr(self, "_h", None) and _lib is not None:
            _lib.or_model_free(self._h)
            self._h = None

    # -- tables --
    def T(self, x, a, y):
        return lib().or_T(self._h, x, a, y)

    def Tprime(self, x, a, k):
        return lib().or_Tprime(self._h, x, a, k)

    def O(self, x, z):
        return lib().or_O(self._h, x, z)

    def R(self, x, a):
        return lib().or_R(self._h, x, a)

    def sig(self, x):
        return lib().or_sig(self._h, x)

    def R_table(self):
        return np.array([[self.R(x, a) for x in range(self.nx)] for a in range(self.na)])

    def O_table(self):
        return np.array([[self.O(x, z) for z in range(self.nz)] for x in range(self.nx)])

    def sig_table(self):
        return np.array([self.sig(x) for x in range(self.nx)], dtype=np.int32)

    # -- belief arithmetic --
    def predict(self, b, a):
        out = np.zeros(self.nx)
        lib().or_predict(self._h, np.ascontiguousarray(b, dtype=np.float64), a, out)
        return out

    def marginal(self, bbar):
        out = np.zeros(self.nz)
        lib().or_marginal(self._h, np.ascontiguousarray(bbar, dtype=np.float64), out)
        return out

    def belief_reward(self, b, a):
        return lib().or_belief_reward(self._h, np.ascontiguousarray(b, dtype=np.float64), a)

    def belief_update(self, b, a, z):
        out = np.zeros(self.nx)
        p = C.c_double(0)
        st = lib().or_belief_update(self._h, np.ascontiguousarray(b, dtype=np.float64), a, z, out, C.byref(p))
        if st != OK:
            raise OracleError(st, "belief_update")
        return out, p.value

    def value_iteration(self, eps=1e-9, max_sweeps=100000):
        V = np.zeros(self.nx)
        Q = np.zeros(self.na * self.nx)
        sw, res = C.c_int(0), C.c_double(0)
        st = lib().or_value_iteration(self._h, eps, max_sweeps, V, Q, C.byref(sw), C.byref(res))
        return st, V, Q.reshape(self.na, self.nx), sw.value, res.value

    def fib(self, eps=1e-9, max_iter=100000):
        alpha = np.zeros(self.na * self.nx)
        it, res = C.c_int(0), C.c_double(0)
        st = lib().or_fib(self._h, eps, max_iter, alpha, C.byref(it), C.byref(res))
        return st, alpha.reshape(self.na, self.nx), it.value, res.value

    def pbvi(self, b0, expansions=3, max_points=16, seed=1, sweeps=30):
        """PBVI lower bound: returns (points [nb][nx], alphas [n][nx], alpha actions)."""
        L = lib()
        h = L.or_pbvi_build(self._h, np.ascontiguousarray(b0, dtype=np.float64), expansions, max_points, seed, sweeps)
        nb, nal = L.or_pbvi_npoints(h), L.or_pbvi_nalpha(h)
        pts = np.zeros((nb, self.nx))
        for i in range(nb):
            L.or_pbvi_point(h, i, pts[i])
        al = np.zeros((nal, self.nx))
        acts = np.zeros(nal, np.int32)
        for i in range(nal):
            a = C.c_int(0)
            L.or_pbvi_alpha(h, i, al[i], C.byref(a))
            acts[i] = a.value
        L.or_pbvi_free(h)
        return pts, al, acts

    def best_first(self, alphaU, alphaL, actL, b0, n, expansions, max_depth=8, gap_tol=0.0, seed=1, step=0,
                   episode=0, mode=MODE_FREQ, sampler=0, replay=None, replay_tol=1e-4):
        """Anytime best-first QVTS (Alg. 1-7, Eq. 8) with U = V_FIB, L = V_PBVI leaves.  Returns a
        dict: action, stop, n_exp, subs, mism, U, L, UQ, LQ, expanded (paths), root_trace
        [(U, L) after k expansions], and per V-node arrays path/depth/f/w/U/L/H/E/expanded."""
        t = BfTree(self, alphaU, alphaL, actL, b0, n, expansions, max_depth, gap_tol, seed, step, episode, mode,
                   sampler, replay, replay_tol)
        out = t.result()
        t.close()
        return out

    def qmdp_value(self, Q, b):
        arg = C.c_int(0)
        v = lib().or_qmdp_value(self._h, np.ascontiguousarray(Q, dtype=np.float64).reshape(-1),
                                np.ascontiguousarray(b, dtype=np.float64), C.byref(arg))
        return v, arg.value

    # -- plan step --
    @staticmethod
    def _cfg(depth, n, seed, step, episode, mode, threads, replay, sampler=0):
        cfg = PlanCfg(depth, n, mode, threads, seed, step, episode, sampler, 0, None, None, None, None)
        keep = None
        if replay:
            # entries (qpath, sample j, GPU z[, GPU state index x]); the ancestral sampler replays x
            rp = np.array([r[0] for r in replay], dtype=np.uint64)
            rj = np.array([r[1] for r in replay], dtype=np.int32)
            rz = np.array([r[2] for r in replay], dtype=np.uint8)
            rx = np.array([r[3] if len(r) > 3 else -1 for r in replay], dtype=np.int32)
            keep = (rp, rj, rz, rx)
            cfg.n_replay = len(replay)
            cfg.replay_path = rp.ctypes.data
            cfg.replay_j = rj.ctypes.data
            cfg.replay_z = rz.ctypes.data
            cfg.replay_x = rx.ctypes.data if any(len(r) > 3 for r in replay) else None
        return cfg, keep

    def plan(self, Q, b0, depth, n, seed=1, step=0, episode=0, mode=MODE_FREQ, trace=False,
             capture_beliefs=False, threads=0, replay=None, sampler=0) -> PlanResult:
        L = lib()
        cfg, _keep = self._cfg(depth, n, seed, step, episode, mode, threads, replay, sampler)
        tr = L.or_trace_new(1 if capture_beliefs else 0) if trace else None
        act = C.c_int(0)
        qroot = np.zeros(self.na)
        st = L.or_plan(self._h, np.ascontiguousarray(Q, dtype=np.float64).reshape(-1),
                       np.ascontiguousarray(b0, dtype=np.float64), C.byref(cfg), C.byref(act), qroot, tr)
        if st != OK:
            if tr:
                L.or_trace_free(tr)
            raise OracleError(st, "plan")
        T = None
        if tr:
            T = self._export(tr)
            L.or_trace_free(tr)
        return PlanResult(act.value, qroot, T)

    def _export(self, tr) -> Trace:
        L = lib()
        nq, nv, ns = L.or_trace_nq(tr), L.or_trace_nv(tr), L.or_trace_nsamples(tr)
        qp = np.zeros(nq, np.uint64); ql = np.zeros(nq, np.int32); qa = np.zeros(nq, np.int32)
        qR = np.zeros(nq); qP = np.zeros(nq * 16); qc = np.zeros(nq * 16, np.uint16); qQ = np.zeros(nq)
        qz = np.zeros(max(1, nq * ns), np.uint8); qf = np.zeros(max(1, nq * ns), np.uint8)
        if nq:
            L.or_trace_export_q(tr, qp, ql, qa, qR, qP, qc, qQ, qz, qf)
        vp = np.zeros(nv, np.uint64); vl = np.zeros(nv, np.int32); vV = np.zeros(nv)
        vz = np.zeros(nv, np.int32); vf = np.zeros(nv, np.int32); vb = np.zeros(nv, np.int64)
        if nv:
            L.or_trace_export_v(tr, vp, vl, vV, vz, vf, vb)
        bel = {}
        for i in range(nv):
            if vb[i] >= 0:
                out = np.zeros(self.nx)
                L.or_trace_belief(tr, int(vb[i]), out)
                bel[int(vp[i])] = out
        return Trace(qp, ql, qa, qR, qP.reshape(nq, 16), qc.reshape(nq, 16), qQ,
                     qz[:nq * ns].reshape(nq, ns), qf[:nq * ns].reshape(nq, ns),
                     vp, vl, vV, vz, vf, bel)

    def qnode_sample(self, b, a, qpath, n, seed=1, step=0, episode=0, sampler=0, replay=None):
        cfg, _keep = self._cfg(0, n, seed, step, episode, MODE_FREQ, 1, replay, sampler)
        P = np.zeros(16); R = C.c_double(0)
        z = np.zeros(n, np.uint8); f = np.zeros(n, np.uint8); cnt = np.zeros(16, np.uint16)
        lib().or_qnode_sample(self._h, np.ascontiguousarray(b, dtype=np.float64), a, int(qpath),
                              C.byref(cfg), P, C.byref(R), z, f, cnt)
        return P, R.value, z, f.astype(bool), cnt

    def vnode_value(self, Q, b, vpath, level, depth, n, seed=1, step=0, episode=0, mode=MODE_FREQ, replay=None):
        cfg, _keep = self._cfg(depth, n, seed, step, episode, mode, 1, replay)
        qv = np.zeros(self.na)
        v = lib().or_vnode_value(self._h, np.ascontiguousarray(Q, dtype=np.float64).reshape(-1),
                                 np.ascontiguousarray(b, dtype=np.float64), int(vpath), level,
                                 C.byref(cfg), qv)
        return v, qv

    # -- episodes & baselines --
    def run_episode(self, Q, b0, planner, depth=3, n=8, max_steps=500, stop_patience=3, seed=1, episode=0):
        cfg = EpisodeCfg(planner, depth, n, max_steps, stop_patience, seed, episode)
        rec = EpisodeRecord()
        la = np.zeros(max_steps, np.int32); lz = np.zeros(max_steps, np.int32); lx = np.zeros(max_steps, np.int32)
        st = lib().or_run_episode(self._h, np.ascontiguousarray(Q, dtype=np.float64).reshape(-1),
                                  np.ascontiguousarray(b0, dtype=np.float64), C.byref(cfg), C.byref(rec),
                                  la, lz, lx)
        if st != OK:
            raise OracleError(st, "run_episode")
        s = rec.steps
        return rec, la[:s].copy(), lz[:s].copy(), lx[:s].copy()

    def astar_action(self, start):
        return lib().or_astar_action(self._h, start)

    def astar_length(self, start):
        return lib().or_astar_length(self._h, start)

    def belief_mode(self, b):
        return lib().or_belief_mode(self._h, np.ascontiguousarray(b, dtype=np.float64))

    def ancestral_sample(self, b, a, ctr, key):
        return lib().or_ancestral_sample(self._h, np.ascontiguousarray(b, dtype=np.float64), a,
                                         np.asarray(ctr, dtype=np.uint32), np.asarray(key, dtype=np.uint32))


def qpath_child(vpath: int, level: int, a_id: int) -> int:
    """Tree path of the Q-node for stencil action a_id under the V-node `vpath` at `level`
    (SURVEY Appendix A.3)."""
    return int(vpath) | ((a_id + 1) << (8 * level))


def vpath_child(qpath: int, level: int, z: int) -> int:
    return int(qpath) | (z << (8 * level + 4))
