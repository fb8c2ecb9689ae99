"""ctypes binding of include/ca.h (argument marshalling only; every step of the
method runs in the CUDA kernels of libca.so).  Fails loudly if the library or a
B200 is missing -- there is no fallback path."""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
# CA_LIBRARY: a tuning variant built by profiles/tune.py (default: the in-tree library)
LIB = os.environ.get("CA_LIBRARY") or os.path.join(HERE, "libca.so")

CA_OK = 0
CA_W_NOT_CONVERGED = 1
CA_W_PAIR_FAILURES = 2
_ERRS = {-1: "CA_E_INVALID", -2: "CA_E_DIM", -3: "CA_E_GEOMETRY", -4: "CA_E_UNSUPPORTED",
         -5: "CA_E_CUDA", -6: "CA_E_NCCL", -7: "CA_E_OOM"}


class CAError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"{_ERRS.get(code, code)}: {msg}")
        self.code = code


class Desc(C.Structure):
    _fields_ = [
        ("dim", C.c_int32), ("n_scenes", C.c_int32), ("horizon", C.c_int32), ("n_state", C.c_int32),
        ("n_ctrl", C.c_int32), ("pose_model", C.c_int32), ("pose_idx", C.c_int32 * 4),
        ("n_parts", C.c_int32), ("part_off", C.c_void_p), ("part_A", C.c_void_p), ("part_b", C.c_void_p),
        ("n_obs", C.c_int32), ("obs_off", C.c_void_p), ("obs_C", C.c_void_p), ("obs_d", C.c_void_p),
        ("dyn_per_scene", C.c_int32), ("dyn_per_time", C.c_int32),
        ("dyn_A", C.c_void_p), ("dyn_B", C.c_void_p), ("dyn_c", C.c_void_p),
        ("Qs", C.c_void_p), ("Qu", C.c_void_p), ("s0", C.c_void_p), ("s_ref", C.c_void_p),
        ("s_init", C.c_void_p),
        ("sigma", C.c_double), ("eps_pri", C.c_double), ("eps_dual", C.c_double), ("max_iters", C.c_int32),
        ("lemke_pivot_tol", C.c_double), ("lemke_tie_tol", C.c_double), ("lemke_max_pivot_factor", C.c_int32),
        ("prox_eps", C.c_double), ("obs_step", C.c_void_p),
        ("workspace", C.c_void_p), ("workspace_bytes", C.c_size_t),
        ("dyn_model", C.c_int32), ("dt", C.c_double),
        ("s_min", C.c_void_p), ("s_max", C.c_void_p), ("u_min", C.c_void_p), ("u_max", C.c_void_p),
        ("box_rho", C.c_double), ("sense_half", C.c_void_p), ("part_ctr", C.c_void_p),
        ("prox_solver", C.c_int32),
    ]


class DistDesc(C.Structure):
    _fields_ = [("world_size", C.c_int32), ("rank", C.c_int32), ("nccl_id", C.c_void_p),
                ("scene_shards", C.c_int32), ("obstacle_shards", C.c_int32)]


RES_FIELDS = ("r_pri", "r_dual", "n_pairs", "n_fail", "pivots", "n_ray", "n_iterlimit", "n_neg_ye", "max_pivots",
              "ms_sweep", "ms_comm", "ms_riccati", "ms_mult")


class Residuals(C.Structure):
    _fields_ = [("r_pri", C.c_double), ("r_dual", C.c_double), ("n_pairs", C.c_int64),
                ("n_fail", C.c_int64), ("pivots", C.c_int64), ("n_ray", C.c_int64), ("n_iterlimit", C.c_int64),
                ("n_neg_ye", C.c_int64), ("max_pivots", C.c_int32), ("reserved_", C.c_int32),
                ("ms_sweep", C.c_float), ("ms_comm", C.c_float), ("ms_riccati", C.c_float), ("ms_mult", C.c_float)]

    def as_dict(self):
        return {f: getattr(self, f) for f in RES_FIELDS}


class SolveReport(C.Structure):
    _fields_ = [("iterations", C.c_int32), ("converged", C.c_int32), ("last", Residuals)]


_lib = None


def library_path() -> str:
    return LIB


def lib():
    """Load libca.so (in-tree).  Raises if it has not been built."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB):
            raise ImportError(f"{LIB} not built: run python -c 'import __graft_entry__ as g; g.build()'")
        L = C.CDLL(LIB)
        vp, dp, i64p = C.c_void_p, C.POINTER(C.c_double), C.POINTER(C.c_int64)
        L.ca_last_error.restype = C.c_char_p
        L.ca_problem_create.argtypes = [C.POINTER(Desc), C.c_int, vp, C.POINTER(vp)]
        L.ca_problem_destroy.argtypes = [vp]
        L.ca_workspace_size.argtypes = [C.POINTER(Desc), vp, C.POINTER(C.c_size_t)]
        L.ca_problem_destroy.restype = None
        L.ca_problem_load.argtypes = [vp, C.POINTER(Desc)]
        L.ca_problem_info.argtypes = [vp, i64p, C.POINTER(C.c_int32), i64p]
        L.ca_scale_detect.argtypes = [vp, vp, vp, vp]
        L.ca_admm_iterate.argtypes = [vp, C.c_int32, vp]
        L.ca_admm_solve.argtypes = [vp, C.POINTER(SolveReport)]
        L.ca_get_solve_scenes.argtypes = [vp, vp, vp]
        L.ca_get_stage_records.argtypes = [vp, vp]
        L.ca_primal_step_records.argtypes = [vp, vp]
        L.ca_dual_sweep.argtypes = [vp, C.POINTER(Residuals)]
        L.ca_primal_step.argtypes = [vp]
        L.ca_multiplier_update.argtypes = [vp, C.POINTER(Residuals)]
        L.ca_get_scene_residuals.argtypes = [vp, vp, vp]
        L.ca_get_trajectory.argtypes = [vp, vp, vp]
        L.ca_get_pair_state.argtypes = [vp, C.c_int64, C.c_int64, vp, vp, vp, vp, vp, vp]
        L.ca_set_iterate.argtypes = [vp, vp, vp, vp, vp, vp]
        if hasattr(L, "ca_get_box_state") or not os.environ.get("CA_LIBRARY"):  # older tuning builds lack it
            L.ca_get_box_state.argtypes = [vp, vp, vp, vp, vp, vp]
            L.ca_get_box_state.restype = C.c_int32
        L.ca_kernel_times.argtypes = [vp, dp, i64p, C.c_int32]
        L.ca_set_timing.argtypes = [vp, C.c_int32]
        L.ca_set_record_basis.argtypes = [vp, C.c_int32]
        L.ca_fp64_peak.argtypes = [C.c_int, C.c_double, dp]
        L.ca_reset_iterate.argtypes = [vp]
        L.ca_debug_trace.argtypes = [vp, C.c_int64, vp]
        L.ca_nccl_unique_id.argtypes = [vp]
        L.ca_obstacle_partition.argtypes = [C.c_int32, C.c_int32, vp, C.c_int32, C.c_int32,
                                            C.POINTER(C.c_int32), C.POINTER(C.c_int32)]
        L.ca_problem_create_dist.argtypes = [C.POINTER(Desc), C.POINTER(DistDesc), C.c_int, vp, C.POINTER(vp)]
        for name in ("ca_problem_create", "ca_problem_load", "ca_problem_info", "ca_scale_detect",
                     "ca_admm_iterate", "ca_admm_solve", "ca_dual_sweep", "ca_primal_step",
                     "ca_multiplier_update", "ca_get_scene_residuals", "ca_get_trajectory",
                     "ca_get_pair_state", "ca_set_iterate", "ca_kernel_times", "ca_set_timing",
                     "ca_set_record_basis", "ca_fp64_peak", "ca_reset_iterate", "ca_debug_trace",
                     "ca_nccl_unique_id", "ca_obstacle_partition", "ca_problem_create_dist", "ca_workspace_size",
                     "ca_get_solve_scenes", "ca_get_stage_records", "ca_primal_step_records"):
            getattr(L, name).restype = C.c_int32
        _lib = L
    return _lib


def _check(rc, ok=(CA_OK, CA_W_PAIR_FAILURES, CA_W_NOT_CONVERGED)):
    if rc not in ok:
        raise CAError(rc, lib().ca_last_error().decode())
    return rc


def _ptr(a):
    return None if a is None else a.ctypes.data


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def _i32(a):
    return np.ascontiguousarray(a, dtype=np.int32)


def make_desc(sc, keep: dict, s_init=None, pivot_tol=0.0, tie_tol=0.0, max_pivot_factor=0, eps_pri=0.0,
              eps_dual=0.0, max_iters=0, prox_eps=0.0, sigma=None, prox_solver=0) -> Desc:
    """Marshal a problem (any object with the attributes of scenes.Scene) into ca_problem_desc."""
    def k(name, arr):
        keep[name] = arr
        return arr.ctypes.data

    D = Desc()
    D.dim, D.n_scenes, D.horizon = sc.dim, sc.n_scenes, sc.horizon
    D.n_state, D.n_ctrl, D.pose_model = sc.n_state, sc.n_ctrl, sc.pose_model
    for a in range(4):
        D.pose_idx[a] = int(sc.pose_idx[a])
    D.n_parts = len(sc.part_off) - 1
    D.part_off = k("part_off", _i32(sc.part_off))
    D.part_A = k("part_A", _f64(sc.part_A))
    D.part_b = k("part_b", _f64(sc.part_b))
    D.n_obs = sc.n_obs
    D.obs_off = k("obs_off", _i32(sc.obs_off))
    D.obs_C = k("obs_C", _f64(sc.obs_C) if sc.obs_C.size else np.zeros((1, sc.dim)))
    D.obs_d = k("obs_d", _f64(sc.obs_d) if sc.obs_d.size else np.zeros(1))
    D.dyn_per_scene, D.dyn_per_time = sc.dyn_per_scene, sc.dyn_per_time
    D.dyn_A = k("dyn_A", _f64(sc.dyn_A))
    D.dyn_B = k("dyn_B", _f64(sc.dyn_B))
    D.dyn_c = k("dyn_c", _f64(sc.dyn_c))
    D.Qs = k("Qs", _f64(sc.Qs))
    D.Qu = k("Qu", _f64(sc.Qu))
    D.s0 = k("s0", _f64(sc.s0))
    D.s_ref = k("s_ref", _f64(sc.s_ref))
    D.s_init = None if s_init is None else k("s_init", _f64(s_init))
    D.sigma = sc.sigma if sigma is None else sigma
    D.eps_pri, D.eps_dual, D.max_iters = eps_pri, eps_dual, max_iters
    D.lemke_pivot_tol, D.lemke_tie_tol, D.lemke_max_pivot_factor = pivot_tol, tie_tol, max_pivot_factor
    D.prox_eps = prox_eps
    D.prox_solver = prox_solver  # NEXT f4: 0 dual Newton, 1 dense Lemke (prox_eps > 0 only)
    step = getattr(sc, "obs_step", None)
    D.obs_step = None if step is None else k("obs_step", _f64(step).reshape(-1, sc.dim))
    D.dyn_model, D.dt = int(getattr(sc, "dyn_model", 0)), float(sc.dt)
    for name, n in (("s_min", sc.n_state), ("s_max", sc.n_state), ("u_min", sc.n_ctrl), ("u_max", sc.n_ctrl)):
        v = getattr(sc, name, None)  # NEXT f1 boxes (None = unbounded)
        setattr(D, name, None if v is None else k(name, _f64(v).reshape(n)))
    D.box_rho = float(getattr(sc, "box_rho", 0.0))
    half = getattr(sc, "sense_half", None)  # NEXT f3 sensing box (None = every obstacle)
    D.sense_half = None if half is None else k("sense_half", _f64(half).reshape(sc.dim))
    ctr = getattr(sc, "part_ctr", None)  # NEXT f3 per-part scaling centres (None = body origin)
    D.part_ctr = None if ctr is None else k("part_ctr", _f64(ctr).reshape(-1, sc.dim))
    return D


class Problem:
    """A batched MPC problem resident on one B200 (ca_problem handle)."""

    def __init__(self, sc, device: int = 0, stream: int | None = None, dist=None, workspace: str | None = None,
                 **params):
        """dist = (world_size, rank, nccl_id bytes[, scene_shards, obstacle_shards]): rank of
        the sharded full problem `sc` (include/ca.h ca_problem_create_dist; grid 0, 0 =
        obstacle sharding only); None = single GPU.
        workspace = "torch": every device buffer is carved out of one torch uint8 tensor
        of ca_workspace_size bytes (device memory owned by PyTorch's allocator)."""
        self.sc = sc
        self.params = params
        self._keep = {}
        desc = make_desc(sc, self._keep, **params)
        h = C.c_void_p()
        self.dist = dist
        if dist is not None:
            world, rank, nid = dist[:3]
            ws, wo = (tuple(dist[3:5]) + (0, 0))[:2]
            self._nid = C.create_string_buffer(bytes(nid), 128)
            dd = DistDesc(world, rank, C.cast(self._nid, C.c_void_p), ws, wo)
        if workspace == "torch":
            import torch

            nbytes = C.c_size_t()
            _check(lib().ca_workspace_size(C.byref(desc), C.byref(dd) if dist is not None else None,
                                           C.byref(nbytes)))
            self._ws = torch.empty(nbytes.value, dtype=torch.uint8, device=torch.device("cuda", device))
            desc.workspace, desc.workspace_bytes = self._ws.data_ptr(), nbytes.value
        elif workspace is not None:
            raise ValueError("workspace must be None or 'torch'")
        if dist is None:
            _check(lib().ca_problem_create(C.byref(desc), device, stream, C.byref(h)), ok=(CA_OK,))
            self.j0, self.j1 = 0, sc.n_obs
        else:
            _check(lib().ca_problem_create_dist(C.byref(desc), C.byref(dd), device, stream, C.byref(h)), ok=(CA_OK,))
            self.grid = grid_position(sc.n_scenes, world, rank, ws, wo)
            b0, b1 = self.grid["scenes"]
            self.j0, self.j1 = obstacle_partition(sc.subset(range(b0, b1)) if (b0, b1) != (0, sc.n_scenes) else sc,
                                                  self.grid["Wo"], self.grid["ro"])
            self.sc = sc.subset(range(b0, b1)) if (b0, b1) != (0, sc.n_scenes) else sc  # the rank's scenes
        self.h = h
        n, ny, nb = C.c_int64(), C.c_int32(), C.c_int64()
        _check(lib().ca_problem_info(h, C.byref(n), C.byref(ny), C.byref(nb)))
        self.n_pairs, self.ny, self.device_bytes = n.value, ny.value, nb.value

    def close(self):
        if getattr(self, "h", None):
            lib().ca_problem_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- per-batch inputs ---------------------------------------------------
    def load(self, sc, **params):
        keep = {}
        desc = make_desc(sc, keep, **{**self.params, **params})
        _check(lib().ca_problem_load(self.h, C.byref(desc)), ok=(CA_OK,))
        self.sc = sc

    def reset_iterate(self):
        _check(lib().ca_reset_iterate(self.h))

    # -- the method -------------------------------------------------------------
    def admm_iterate(self, iters: int, hist: bool = True):
        H = (Residuals * iters)() if hist else None
        rc = _check(lib().ca_admm_iterate(self.h, iters, H))
        if not hist:
            return rc
        return rc, {f: np.array([getattr(r, f) for r in H]) for f in RES_FIELDS}

    def admm_solve(self):
        """ADMM until Eq. 18 per scene (include/ca.h ca_admm_solve): (rc, report dict,
        per-scene iterations, per-scene converged flags)."""
        rep = SolveReport()
        rc = _check(lib().ca_admm_solve(self.h, C.byref(rep)))
        B = self.sc.n_scenes
        it = np.empty(B, np.int32)
        cv = np.empty(B, np.int32)
        _check(lib().ca_get_solve_scenes(self.h, _ptr(it), _ptr(cv)))
        out = {"iterations": rep.iterations, "converged": bool(rep.converged), **rep.last.as_dict()}
        return rc, out, it, cv.astype(bool)

    def dual_sweep(self):
        r = Residuals()
        rc = _check(lib().ca_dual_sweep(self.h, C.byref(r)))
        return rc, r

    def primal_step(self):
        _check(lib().ca_primal_step(self.h))

    def stage_records(self):
        """[B, N, R] per-(scene, t) records of the last dual sweep (include/ca.h)."""
        sc = self.sc
        R = rec_len(sc.dim)
        out = np.empty((sc.n_scenes, sc.horizon, R))
        _check(lib().ca_get_stage_records(self.h, _ptr(out)))
        return out

    def primal_step_records(self, rec):
        rec = _f64(rec)
        _check(lib().ca_primal_step_records(self.h, _ptr(rec)))

    def multiplier_update(self):
        r = Residuals()
        _check(lib().ca_multiplier_update(self.h, C.byref(r)))
        return r

    def scale_detect(self, states=None, want_alpha=True):
        st = None if states is None else _f64(states)
        alpha = np.empty(max(self.n_pairs, 1)) if want_alpha else None
        amin = np.empty(self.sc.n_scenes)
        _check(lib().ca_scale_detect(self.h, _ptr(st), _ptr(alpha), _ptr(amin)))
        return alpha, amin

    # -- state --------------------------------------------------------------
    def trajectory(self):
        sc = self.sc
        s = np.empty((sc.n_scenes, sc.horizon + 1, sc.n_state))
        u = np.empty((sc.n_scenes, sc.horizon, sc.n_ctrl))
        _check(lib().ca_get_trajectory(self.h, _ptr(s), _ptr(u)))
        return s, u

    def scene_residuals(self):
        rp = np.empty(self.sc.n_scenes)
        rd = np.empty(self.sc.n_scenes)
        _check(lib().ca_get_scene_residuals(self.h, _ptr(rp), _ptr(rd)))
        return rp, rd

    def pair_state(self, p0: int = 0, count: int | None = None, zmask: bool = False, fields=None):
        """Pair state of pairs [p0, p0 + count): y, zeta, xi, pivots, status (and zmask);
        `fields` restricts the copies (e.g. ("status",) for a cheap failure scan)."""
        count = self.n_pairs - p0 if count is None else count
        d = self.sc.dim
        want = set(fields) if fields is not None else {"y", "zeta", "xi", "pivots", "status"} | ({"zmask"} if zmask else set())
        shapes = {"y": ((count, self.ny), np.float64), "zeta": ((count,), np.float64), "xi": ((count, d), np.float64),
                  "pivots": ((count,), np.int32), "status": ((count,), np.int32), "zmask": ((count,), np.uint32)}
        out = {k: np.empty(*shapes[k]) for k in want}
        _check(lib().ca_get_pair_state(self.h, p0, count, *[_ptr(out.get(k)) for k in
                                                              ("y", "zeta", "xi", "pivots", "status", "zmask")]))
        return out

    def set_iterate(self, s=None, u=None, y=None, zeta=None, xi=None):
        arrs = [None if a is None else _f64(a) for a in (s, u, y, zeta, xi)]
        if arrs[2] is not None:
            assert arrs[2].shape == (self.n_pairs, self.ny), arrs[2].shape
        _check(lib().ca_set_iterate(self.h, *[_ptr(a) for a in arrs]))

    def box_state(self):
        """(w_s, l_s, w_u, l_u, res) of the box block (NEXT f1)."""
        sc = self.sc
        ws, ls = np.empty((sc.n_scenes, sc.horizon + 1, sc.n_state)), np.empty((sc.n_scenes, sc.horizon + 1, sc.n_state))
        wu, lu = np.empty((sc.n_scenes, sc.horizon, sc.n_ctrl)), np.empty((sc.n_scenes, sc.horizon, sc.n_ctrl))
        res = np.empty(sc.n_scenes)
        _check(lib().ca_get_box_state(self.h, *[_ptr(a) for a in (ws, ls, wu, lu, res)]))
        return ws, ls, wu, lu, res

    def debug_trace(self, p: int = -1):
        out = np.empty((64, 48))
        _check(lib().ca_debug_trace(self.h, p, _ptr(out)))
        return out

    def set_timing(self, on: bool = True):
        _check(lib().ca_set_timing(self.h, int(on)))

    def set_record_basis(self, on: bool = True):
        _check(lib().ca_set_record_basis(self.h, int(on)))

    def kernel_times(self, reset: bool = False):
        """{family: (device ms, count)}: the library's kernel families and 'comm' (NCCL)."""
        ms = (C.c_double * 6)()
        ln = (C.c_int64 * 6)()
        _check(lib().ca_kernel_times(self.h, ms, ln, int(reset)))
        names = ("sweep", "primal", "multiplier", "scale", "other", "comm")
        return {n: (ms[i], ln[i]) for i, n in enumerate(names)}


def nccl_unique_id() -> bytes:
    buf = C.create_string_buffer(128)
    _check(lib().ca_nccl_unique_id(buf))
    return buf.raw


def rec_len(d: int) -> int:
    """doubles per record: (d+1)(d+2)/2 + (d+1) Gauss-Newton terms + 8 statistics"""
    return (d + 1) * (d + 2) // 2 + (d + 1) + 8


def grid_position(n_scenes: int, world: int, rank: int, scene_shards: int = 0, obstacle_shards: int = 0):
    """The rank's place in the scene x obstacle grid (include/ca.h ca_dist_desc; the
    library computes the same on its side): shard indices and the scene block."""
    ws, wo = scene_shards, obstacle_shards
    if ws <= 0 and wo <= 0:
        ws, wo = 1, world
    elif ws <= 0:
        ws = world // wo
    elif wo <= 0:
        wo = world // ws
    rs, ro = rank // wo, rank % wo
    return {"Ws": ws, "Wo": wo, "rs": rs, "ro": ro,
            "scenes": (n_scenes * rs // ws, n_scenes * (rs + 1) // ws)}


def obstacle_partition(sc, world: int, rank: int):
    """[j0, j1): the obstacle block of `rank` in an obstacle-sharded run (host only)."""
    off = _i32(sc.obs_off)
    j0, j1 = C.c_int32(), C.c_int32()
    _check(lib().ca_obstacle_partition(sc.n_scenes, sc.n_obs, off.ctypes.data, world, rank, C.byref(j0),
                                       C.byref(j1)))
    return j0.value, j1.value


def fp64_peak(device: int = 0, ms: float = 200.0) -> float:
    t = C.c_double()
    _check(lib().ca_fp64_peak(device, ms, C.byref(t)))
    return t.value
