"""ctypes wrapper of the plain-C CPU oracle (oracle/orc.c).

TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference legs may import this package.  It shares no
code with the product package paper_2406_07048_b200/ and never imports it.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(HERE, "liborc.so")

OK, RAY, ITER_LIMIT, NEG_YE = 0, 1, 2, 3


def build(force: bool = False) -> str:
    src = os.path.join(HERE, "orc.c")
    if force or not os.path.exists(LIB) or os.path.getmtime(LIB) < max(
        os.path.getmtime(src), os.path.getmtime(os.path.join(HERE, "orc.h"))
    ):
        subprocess.check_call(
            ["gcc", "-O2", "-std=c11", "-ffp-contract=off", "-fno-fast-math", "-fPIC", "-shared", "-pthread",
             "-o", LIB, src, "-lm"]
        )
    return LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        _lib = C.CDLL(LIB)
        dp, ip = C.POINTER(C.c_double), C.POINTER(C.c_int)
        _lib.orc_pose.argtypes = [C.c_int, ip, C.c_int, dp, dp, dp]
        _lib.orc_scale_lp.argtypes = [C.c_int, C.c_int, dp, dp, dp, dp, C.c_int, dp, dp, dp, dp]
        _lib.orc_scale_lp.restype = C.c_int
        _lib.orc_build_K.argtypes = [C.c_int, C.c_int, dp, C.c_int, dp, dp, dp, dp, dp]
        _lib.orc_pair_lcp.argtypes = [C.c_int, C.c_int, dp, dp, C.c_int, dp, dp, dp, dp, C.c_double,
                                      dp, C.c_double, dp, dp, dp, ip, dp, dp]
        _lib.orc_lemke.argtypes = [C.c_int, dp, dp, C.c_double, C.c_double, C.c_int, dp, ip, ip]
        _lib.orc_lemke.restype = C.c_int
        _lib.orc_pair_solve.argtypes = [C.c_int, C.c_int, dp, dp, C.c_int, dp, dp, dp, dp, C.c_double,
                                        dp, C.c_double, dp, C.c_double, C.c_double, C.c_int, dp, ip, ip]
        _lib.orc_pair_solve.restype = C.c_int
        _lib.orc_init_iterate.argtypes = [C.c_void_p, C.c_void_p]
        _lib.orc_reset_box.argtypes = [C.c_void_p, C.c_void_p]
        _lib.orc_sense.argtypes = [C.c_void_p, dp, C.c_void_p]
        _lib.orc_dual_sweep.argtypes = [C.c_void_p, C.c_void_p, dp]
        _lib.orc_dual_sweep.restype = C.c_longlong
        _lib.orc_primal_step.argtypes = [C.c_void_p, C.c_void_p]
        _lib.orc_primal_step.restype = C.c_int
        _lib.orc_multiplier_update.argtypes = [C.c_void_p, C.c_void_p, dp]
        _lib.orc_admm_iterate.argtypes = [C.c_void_p, C.c_void_p, C.c_int, dp, dp]
        _lib.orc_admm_iterate.restype = C.c_longlong
        _lib.orc_scale_detect.argtypes = [C.c_void_p, dp, dp]
        _lib.orc_scale_detect.restype = C.c_longlong
        _lib.orc_check_stopping.argtypes = [C.c_double, C.c_double, C.c_double, C.c_double]
        _lib.orc_check_stopping.restype = C.c_int
        _lib.orc_admm_solve.argtypes = [C.c_void_p, C.c_void_p, C.c_double, C.c_double, C.c_int, ip, ip, dp, dp]
        _lib.orc_admm_solve.restype = C.c_longlong
        _lib.orc_admm_iterate_mt.argtypes = [C.c_void_p, C.c_void_p, C.c_int, dp, dp, C.c_int]
        _lib.orc_admm_iterate_mt.restype = C.c_longlong
    return _lib


def _d(a):
    return a.ctypes.data_as(C.POINTER(C.c_double))


def _i(a):
    return a.ctypes.data_as(C.POINTER(C.c_int))


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def _i32(a):
    return np.ascontiguousarray(a, dtype=np.int32)


class _Problem(C.Structure):
    _fields_ = [
        ("dim", C.c_int), ("n_scenes", C.c_int), ("horizon", C.c_int), ("n_state", C.c_int),
        ("n_ctrl", C.c_int), ("pose_model", C.c_int), ("pose_idx", C.c_int * 4),
        ("n_parts", C.c_int), ("part_off", C.c_void_p), ("part_A", C.c_void_p), ("part_b", C.c_void_p),
        ("n_obs", C.c_int), ("obs_off", C.c_void_p), ("obs_C", C.c_void_p), ("obs_d", C.c_void_p),
        ("dyn_per_scene", C.c_int), ("dyn_per_time", C.c_int),
        ("dyn_A", C.c_void_p), ("dyn_B", C.c_void_p), ("dyn_c", C.c_void_p),
        ("Qs", C.c_void_p), ("Qu", C.c_void_p), ("s0", C.c_void_p), ("s_ref", C.c_void_p),
        ("sigma", C.c_double), ("pivot_tol", C.c_double), ("tie_tol", C.c_double),
        ("max_pivot_factor", C.c_int), ("ny", C.c_int), ("prox_eps", C.c_double), ("obs_step", C.c_void_p),
        ("dyn_model", C.c_int), ("dt", C.c_double),
        ("s_min", C.c_void_p), ("s_max", C.c_void_p), ("u_min", C.c_void_p), ("u_max", C.c_void_p),
        ("box_rho", C.c_double), ("sensed", C.c_void_p), ("part_ctr", C.c_void_p),
    ]


class _Iterate(C.Structure):
    _fields_ = [("s", C.c_void_p), ("u", C.c_void_p), ("y", C.c_void_p), ("zeta", C.c_void_p),
                ("xi", C.c_void_p), ("pivots", C.c_void_p), ("status", C.c_void_p),
                ("ws", C.c_void_p), ("ls", C.c_void_p), ("wu", C.c_void_p), ("lu", C.c_void_p),
                ("boxres", C.c_void_p), ("zmask", C.c_void_p)]


class Oracle:
    """One batched problem (a scenes.Scene) plus its ADMM iterate, on the CPU."""

    def __init__(self, sc, pivot_tol=1e-11, tie_tol=1e-9, max_pivot_factor=50, sigma=None, prox_eps=0.0):
        self.sc = sc
        self.keep = {}

        def k(name, arr):
            self.keep[name] = arr
            return arr.ctypes.data

        P = _Problem()
        P.dim, P.n_scenes, P.horizon = sc.dim, sc.n_scenes, sc.horizon
        P.n_state, P.n_ctrl, P.pose_model = sc.n_state, sc.n_ctrl, sc.pose_model
        for a in range(4):
            P.pose_idx[a] = int(sc.pose_idx[a])
        P.n_parts = sc.n_parts
        P.part_off = k("part_off", _i32(sc.part_off))
        P.part_A = k("part_A", _f64(sc.part_A))
        P.part_b = k("part_b", _f64(sc.part_b))
        P.n_obs = sc.n_obs
        P.obs_off = k("obs_off", _i32(sc.obs_off))
        P.obs_C = k("obs_C", _f64(sc.obs_C).reshape(-1, sc.dim) if sc.obs_C.size else np.zeros((1, sc.dim)))
        P.obs_d = k("obs_d", _f64(sc.obs_d) if sc.obs_d.size else np.zeros(1))
        P.dyn_per_scene, P.dyn_per_time = sc.dyn_per_scene, sc.dyn_per_time
        P.dyn_A = k("dyn_A", _f64(sc.dyn_A))
        P.dyn_B = k("dyn_B", _f64(sc.dyn_B))
        P.dyn_c = k("dyn_c", _f64(sc.dyn_c))
        P.Qs = k("Qs", _f64(sc.Qs))
        P.Qu = k("Qu", _f64(sc.Qu))
        P.s0 = k("s0", _f64(sc.s0))
        P.s_ref = k("s_ref", _f64(sc.s_ref))
        P.sigma = sc.sigma if sigma is None else sigma
        P.pivot_tol, P.tie_tol, P.max_pivot_factor = pivot_tol, tie_tol, max_pivot_factor
        P.prox_eps = prox_eps
        step = getattr(sc, "obs_step", None)  # NEXT f3: moving obstacles (None = static)
        P.obs_step = None if step is None else k("obs_step", _f64(step).reshape(-1, sc.dim))
        P.dyn_model, P.dt = int(getattr(sc, "dyn_model", 0)), float(sc.dt)  # NEXT f2: SQP relinearisation
        for name, n in (("s_min", sc.n_state), ("s_max", sc.n_state), ("u_min", sc.n_ctrl), ("u_max", sc.n_ctrl)):
            v = getattr(sc, name, None)  # NEXT f1: boxes of Eq. 13c-d (None = unbounded)
            setattr(P, name, None if v is None else k(name, _f64(v).reshape(n)))
        P.box_rho = float(getattr(sc, "box_rho", 0.0))
        ctr = getattr(sc, "part_ctr", None)  # NEXT f3: per-part scaling centres (None = body origin)
        P.part_ctr = None if ctr is None else k("part_ctr", _f64(ctr).reshape(-1, sc.dim))
        self.sensed = None  # NEXT f3 sensing: obstacles meeting the box rho(s0) + [-h, h]
        half = getattr(sc, "sense_half", None)
        if half is not None and sc.n_obs > 0:
            self.sensed = np.zeros(sc.n_scenes * sc.n_obs, np.uint8)
            lib().orc_sense(C.byref(P), _d(_f64(half).reshape(sc.dim)), self.sensed.ctypes.data)
            P.sensed = self.sensed.ctypes.data
        self.ny = P.ny = sc.n_max if sc.n_obs > 0 else 1
        self.P = P
        B, N, ns, nu, d = sc.n_scenes, sc.horizon, sc.n_state, sc.n_ctrl, sc.dim
        npair = sc.n_pairs
        self.s = np.zeros((B, N + 1, ns))
        self.u = np.zeros((B, N, nu))
        self.y = np.zeros((max(npair, 1), self.ny))
        self.zeta = np.zeros(max(npair, 1))
        self.xi = np.zeros((max(npair, 1), d))
        self.pivots = np.zeros(max(npair, 1), np.int32)
        self.status = np.zeros(max(npair, 1), np.int32)
        self.ws, self.ls = np.zeros((B, N + 1, ns)), np.zeros((B, N + 1, ns))  # box block (reading #7)
        self.wu, self.lu = np.zeros((B, N, nu)), np.zeros((B, N, nu))
        self.boxres = np.zeros(B)
        self.zmask = np.zeros(max(npair, 1), np.uint32)  # final Lemke basis per pair (last dual sweep)
        It = _Iterate()
        It.s, It.u, It.y = self.s.ctypes.data, self.u.ctypes.data, self.y.ctypes.data
        It.zeta, It.xi = self.zeta.ctypes.data, self.xi.ctypes.data
        It.pivots, It.status = self.pivots.ctypes.data, self.status.ctypes.data
        It.ws, It.ls, It.wu, It.lu = (a.ctypes.data for a in (self.ws, self.ls, self.wu, self.lu))
        It.boxres = self.boxres.ctypes.data
        It.zmask = self.zmask.ctypes.data
        self.I = It
        self.init_iterate()

    def _pp(self):
        return C.byref(self.P), C.byref(self.I)

    def init_iterate(self):
        lib().orc_init_iterate(*self._pp())

    def set_iterate(self, s=None, u=None, y=None, zeta=None, xi=None):
        for name, val in (("s", s), ("u", u), ("y", y), ("zeta", zeta), ("xi", xi)):
            if val is not None:
                getattr(self, name)[...] = np.asarray(val, np.float64).reshape(getattr(self, name).shape)
        lib().orc_reset_box(*self._pp())  # w = Pi_box(s, u), l = 0 (reading #7)

    def dual_sweep(self):
        rd = np.zeros(self.sc.n_scenes)
        fails = lib().orc_dual_sweep(*self._pp(), _d(rd))
        return rd, fails

    def primal_step(self):
        rc = lib().orc_primal_step(*self._pp())
        if rc != 0:
            raise RuntimeError("oracle primal step: condensed Hessian not SPD")

    def multiplier_update(self):
        rp = np.zeros(self.sc.n_scenes)
        lib().orc_multiplier_update(*self._pp(), _d(rp))
        return rp

    def admm_iterate(self, K):
        B = self.sc.n_scenes
        hp = np.zeros((K, B))
        hd = np.zeros((K, B))
        fails = lib().orc_admm_iterate(*self._pp(), K, _d(hp), _d(hd))
        if fails < 0:
            raise RuntimeError("oracle primal step failed")
        return hp, hd, fails

    def admm_iterate_mt(self, K, nthreads):
        """The same K iterations fanned out over nthreads POSIX threads (timing of the
        all-core CPU baseline): over scenes when there are >= nthreads of them (bitwise
        = admm_iterate), else over the pairs of each dual step."""
        B = self.sc.n_scenes
        hp = np.zeros((K, B))
        hd = np.zeros((K, B))
        fails = lib().orc_admm_iterate_mt(*self._pp(), K, _d(hp), _d(hd), int(nthreads))
        if fails < 0:
            raise RuntimeError("oracle primal step failed")
        return hp, hd, fails

    def admm_solve(self, eps_pri, eps_dual, max_iters):
        """ADMM until Eq. 18 per scene, or max_iters: (iters[B], converged[B],
        r_pri[B], r_dual[B], failed pair solves)."""
        B = self.sc.n_scenes
        it = np.zeros(B, np.int32)
        cv = np.zeros(B, np.int32)
        rp = np.zeros(B)
        rd = np.zeros(B)
        fails = lib().orc_admm_solve(*self._pp(), float(eps_pri), float(eps_dual), int(max_iters), _i(it), _i(cv),
                                     _d(rp), _d(rd))
        if fails < 0:
            raise RuntimeError("oracle primal step failed")
        return it, cv.astype(bool), rp, rd, fails

    def scale_detect(self, s=None):
        s = self.s if s is None else _f64(s)
        alpha = np.zeros(max(self.sc.n_pairs, 1))
        lib().orc_scale_detect(C.byref(self.P), _d(s), _d(alpha))
        return alpha[: self.sc.n_pairs]


# --------------------------------------------------------------------------
# single-pair entry points (used by the pins)
# --------------------------------------------------------------------------

def check_stopping(r_pri, r_dual, eps_pri, eps_dual) -> bool:
    """Eq. 18: r_pri <= eps_pri and r_dual <= eps_dual."""
    return bool(lib().orc_check_stopping(float(r_pri), float(r_dual), float(eps_pri), float(eps_dual)))


def pose(model, idx, d, s):
    R = np.zeros(d * d)
    rho = np.zeros(d)
    idx = _i32(list(idx) + [0] * (4 - len(idx)))
    s = _f64(s)
    lib().orc_pose(model, _i(idx), d, _d(s), _d(R), _d(rho))
    return R.reshape(d, d), rho


def scale_lp(A, b, R, rho, Cm, dv):
    A, b, R, rho, Cm, dv = map(_f64, (A, b, R, rho, Cm, dv))
    d = A.shape[1]
    alpha = np.zeros(1)
    y = np.zeros(d)
    rc = lib().orc_scale_lp(d, A.shape[0], _d(A), _d(b), _d(R), _d(rho), Cm.shape[0], _d(Cm), _d(dv),
                            _d(alpha), _d(y))
    if rc != 0:
        raise ValueError("scale LP infeasible")
    return float(alpha[0]), y


def pair_lcp(A, b, Cm, dv, R, rho, zeta, xi, prox_eps=0.0, y_prev=None):
    A, b, Cm, dv, R, rho, xi = map(_f64, (A, b, Cm, dv, R, rho, xi))
    d = A.shape[1]
    nr, no = A.shape[0], Cm.shape[0]
    n = nr + no + 1
    y_prev = _f64(np.zeros(n) if y_prev is None else y_prev)
    K = np.zeros((n, d + 1))
    bvec = np.zeros(d + 1)
    e = np.zeros(1, np.int32)
    M = np.zeros((n, n))
    q = np.zeros(n)
    lib().orc_pair_lcp(d, nr, _d(A), _d(b), no, _d(Cm), _d(dv), _d(R), _d(rho), float(zeta), _d(xi),
                       float(prox_eps), _d(y_prev), _d(K), _d(bvec), _i(e), _d(M), _d(q))
    return K, bvec, int(e[0]), M, q


def lemke(M, q, pivot_tol=1e-11, tie_tol=1e-9, max_pivots=None):
    M, q = _f64(M), _f64(q)
    n = len(q)
    z = np.zeros(n)
    basis = np.zeros(n, np.int32)
    piv = np.zeros(1, np.int32)
    st = lib().orc_lemke(n, _d(M), _d(q), pivot_tol, tie_tol, 50 * n if max_pivots is None else max_pivots,
                         _d(z), _i(basis), _i(piv))
    return z, st, int(piv[0]), basis


def pair_solve(A, b, Cm, dv, R, rho, zeta, xi, pivot_tol=1e-11, tie_tol=1e-9, max_pivot_factor=50,
               prox_eps=0.0, y_prev=None):
    A, b, Cm, dv, R, rho, xi = map(_f64, (A, b, Cm, dv, R, rho, xi))
    d = A.shape[1]
    nr, no = A.shape[0], Cm.shape[0]
    n = nr + no + 1
    y_prev = _f64(np.zeros(n) if y_prev is None else y_prev)
    y = np.zeros(n)
    piv = np.zeros(1, np.int32)
    basis = np.zeros(n, np.int32)
    st = lib().orc_pair_solve(d, nr, _d(A), _d(b), no, _d(Cm), _d(dv), _d(R), _d(rho), float(zeta), _d(xi),
                              float(prox_eps), _d(y_prev), pivot_tol, tie_tol, max_pivot_factor, _d(y), _i(piv), _i(basis))
    return y, st, int(piv[0]), basis
