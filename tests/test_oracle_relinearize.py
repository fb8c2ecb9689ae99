"""Oracle pin for the per-iteration SQP relinearisation (NEXT f2):
with dyn_model = 1 the primal step linearises the unicycle at the current iterate.
Pinned against the same primal step with the LTV model written out independently
(scenes.unicycle_ltv, numpy) at that iterate, and against the plant: the linear
model reproduces the nonlinear one-step map at the linearisation point."""
import dataclasses

import numpy as np

import oracle
import scenes


def test_relinearised_primal_step_equals_explicit_ltv():
    sc = scenes.make_config(7)
    o = oracle.Oracle(sc)
    o.admm_iterate(4)
    o.dual_sweep()
    s_k, u_k = o.s.copy(), o.u.copy()
    A, B, c = scenes.unicycle_ltv(s_k[0, :sc.horizon], sc.dt)
    lin = dataclasses.replace(sc, dyn_model=0, dyn_per_scene=0, dyn_per_time=1, dyn_A=A, dyn_B=B, dyn_c=c)
    ref = oracle.Oracle(lin)
    ref.set_iterate(o.s, o.u, o.y, o.zeta, o.xi)
    o.primal_step()
    ref.primal_step()
    scale = 1.0 + np.abs(ref.s).max()
    assert np.abs(o.s - ref.s).max() <= 1e-10 * scale
    assert np.abs(o.u - ref.u).max() <= 1e-10 * (1.0 + np.abs(ref.u).max())
    assert not np.allclose(s_k, o.s)  # the step moved the trajectory


def test_linear_model_matches_plant_at_linearisation_point():
    rng = np.random.default_rng(7)
    s = np.stack([rng.uniform(-5, 5, 20), rng.uniform(-5, 5, 20), rng.uniform(-3, 3, 20), rng.uniform(0, 10, 20)], 1)
    u = rng.uniform(-1, 1, (20, 2))
    A, B, c = scenes.unicycle_ltv(s)
    dt = scenes.DT
    f = s + dt * np.stack([s[:, 3] * np.cos(s[:, 2]), s[:, 3] * np.sin(s[:, 2]), u[:, 1], u[:, 0]], 1)
    lin = np.einsum("tij,tj->ti", A, s) + np.einsum("tij,tj->ti", B, u) + c
    assert np.abs(f - lin).max() <= 1e-12 * (1.0 + np.abs(f).max())
