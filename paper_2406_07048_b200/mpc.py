"""Receding-horizon closed loop around the ADMM solver.

The paper deploys the method as an MPC loop (0.1 s steps; P:272 and
P:349-351: the dynamics are linearised around the current iterate).  Each MPC step
here:

1. measures the true state s_now (a nonlinear unicycle, the car of C1/C2/C4),
2. re-centres the straight-line reference on it and linearises the dynamics around
   the previous solution shifted by one step (reading #8: the LTV model is held
   fixed within a solve),
3. loads the new problem into the SAME device handle (ca_problem_load), warm-starts
   it with the previous iterate shifted by one timestep (s, u, and every pair's
   y, zeta, xi) via ca_set_iterate,
4. runs K ADMM iterations on the GPU and applies the first control to the plant
   (saturated to the control box, if the problem has one: the ADMM iterate meets the
   box only at convergence, reading #7).

Moving obstacles (obs_step) advance with the loop.  Everything numerical in a solve
runs in libca.so; this module only prepares inputs (host numpy).  The solver is
pluggable (the tests drive the same loop with the CPU oracle for parity).
"""
from __future__ import annotations

import dataclasses
import time

import numpy as np

import scenes


def unicycle_step(s: np.ndarray, u: np.ndarray, dt: float = scenes.DT) -> np.ndarray:
    """The plant: s' = s + dt (v cos th, v sin th, omega, a), u = (a, omega)."""
    x, y, th, v = s
    a, om = u
    return np.array([x + dt * v * np.cos(th), y + dt * v * np.sin(th), th + dt * om, v + dt * a])


def shift_pairs(arr: np.ndarray, sc) -> np.ndarray:
    """Pair arrays (index p = ((b N + t-1) n_parts + i) M + j) shifted by one timestep;
    the last timestep is repeated."""
    B, N, G = sc.n_scenes, sc.horizon, sc.n_parts * sc.n_obs
    a = arr.reshape((B, N, G) + arr.shape[1:])
    out = np.concatenate([a[:, 1:], a[:, -1:]], axis=1)
    return np.ascontiguousarray(out.reshape(arr.shape))


class GpuSolver:
    """The default solver: one device handle, reloaded every MPC step."""

    def __init__(self, **params):
        self.params = params
        self.g = None

    def load(self, sc):
        from . import Problem

        if self.g is None:
            self.g = Problem(sc, **self.params)
        else:
            self.g.load(sc)

    def set_iterate(self, s, u, y, zeta, xi):
        self.g.set_iterate(s, u, y, zeta, xi)

    def admm_iterate(self, K):
        self.g.admm_iterate(K, hist=False)

    def state(self):
        s, u = self.g.trajectory()
        st = self.g.pair_state()
        return s, u, st["y"], st["zeta"], st["xi"]


class RecedingHorizon:
    """Closed loop for a single-scene car problem `sc` (SE2 unicycle, pose (x, y, th)).

    solver: an object with load(scene) / set_iterate(s, u, y, zeta, xi) /
    admm_iterate(K) / state() -> (s, u, y, zeta, xi); default GpuSolver."""

    def __init__(self, sc, K: int, speed: float, lane_y: float = 0.0, solver=None):
        assert sc.n_scenes == 1 and sc.pose_model == scenes.POSE_SE2 and sc.n_state == 4
        self.sc0, self.K, self.speed, self.lane_y = sc, K, speed, lane_y
        self.solver = solver if solver is not None else GpuSolver()
        self.k = 0
        self.s_now = np.asarray(sc.s0[0], float).copy()
        self.prev = None  # (s, u, y, zeta, xi) of the last solve
        self.latency = []

    def reference(self) -> np.ndarray:
        N, dt = self.sc0.horizon, self.sc0.dt
        t = np.arange(N + 1) * dt
        return np.stack([self.s_now[0] + self.speed * t, np.full(N + 1, self.lane_y), np.zeros(N + 1),
                         np.full(N + 1, self.speed)], 1)

    def scene_at(self, s_bar: np.ndarray) -> "scenes.Scene":
        sc, N, dt = self.sc0, self.sc0.horizon, self.sc0.dt
        A, B, c = scenes.unicycle_ltv(s_bar[:N], dt)
        obs_d = sc.obs_d
        if sc.obs_step is not None and self.k:  # obstacles have moved k steps
            disp = np.repeat(sc.obs_step, np.diff(sc.obs_off), axis=0) * self.k
            obs_d = sc.obs_d + np.einsum("ij,ij->i", sc.obs_C, disp)
        return dataclasses.replace(sc, s0=self.s_now[None].copy(), s_ref=self.reference()[None], dyn_per_scene=0,
                                   dyn_per_time=1, dyn_A=A, dyn_B=B, dyn_c=c, obs_d=obs_d)

    def step(self):
        """One MPC step; returns the control applied."""
        if self.prev is None:
            s_bar = self.reference()
        else:
            s_prev, u_prev = self.prev[0], self.prev[1]
            s_bar = np.concatenate([s_prev[1:], unicycle_step(s_prev[-1], u_prev[-1])[None]])
        s_bar[0] = self.s_now
        sc = self.scene_at(s_bar)
        t0 = time.perf_counter()
        self.solver.load(sc)
        if self.prev is not None:
            s_prev, u_prev, y, zeta, xi = self.prev
            s_w = np.concatenate([s_prev[1:], s_prev[-1:]])
            s_w[0] = self.s_now
            u_w = np.concatenate([u_prev[1:], u_prev[-1:]])
            self.solver.set_iterate(s_w[None], u_w[None], shift_pairs(y, sc), shift_pairs(zeta, sc),
                                    shift_pairs(xi, sc))
        self.solver.admm_iterate(self.K)
        s, u, y, zeta, xi = self.solver.state()
        self.latency.append(time.perf_counter() - t0)
        self.prev = (np.array(s[0]), np.array(u[0]), np.array(y), np.array(zeta), np.array(xi))
        u0 = np.array(u[0, 0])
        if self.sc0.u_min is not None or self.sc0.u_max is not None:  # actuator saturation (NEXT f1 boxes)
            u0 = np.clip(u0, self.sc0.u_min if self.sc0.u_min is not None else -np.inf,
                         self.sc0.u_max if self.sc0.u_max is not None else np.inf)
        self.s_now = unicycle_step(self.s_now, u0, self.sc0.dt)
        self.k += 1
        return u0
