"""Oracle pins for moving obstacles (obstacle model of P:208-212 with
a per-timestep offset): obstacle j at timestep t is {x : C_j x <= d_j + t C_j step_j}.

The oracle implements it by shifting the robot's origin (rho - t*step_j, translation
invariance); these tests write the moving obstacle out independently -- as a static
obstacle with shifted offsets d_j + t C_j step_j -- and check every pair's dual step,
multiplier update and scale factor against it.  A scene with all steps zero must equal
the static scene bitwise.
"""
import dataclasses

import numpy as np

import oracle
import scenes
from parity_util import pair_geometry


def moving_scene():
    sc = scenes.make_config(6)
    # keep the test fast: the 12 obstacles nearest to the ego's path, N = 12
    keep = list(range(12))
    M = sc.n_obs
    offs, Cs, ds = [0], [], []
    for j in keep:
        lo, hi = sc.obs_off[j], sc.obs_off[j + 1]
        Cs.append(sc.obs_C[lo:hi])
        ds.append(sc.obs_d[lo:hi])
        offs.append(offs[-1] + hi - lo)
    N = 12
    return dataclasses.replace(
        sc, n_obs=len(keep), horizon=N, obs_off=np.asarray(offs, np.int32), obs_C=np.concatenate(Cs),
        obs_d=np.concatenate(ds), obs_step=np.ascontiguousarray(sc.obs_step[keep]),
        dyn_A=sc.dyn_A[:N], dyn_B=sc.dyn_B[:N], dyn_c=sc.dyn_c[:N], s_ref=sc.s_ref[:, :N + 1])


def shifted(sc, p):
    """Pair p of a moving scene written as a static obstacle at timestep t."""
    b, t, A, bb, Cm, dv = pair_geometry(sc, p)
    j = p % sc.n_obs
    step = sc.obs_step[b * sc.n_obs + j]
    return b, t, A, bb, Cm, dv + t * (Cm @ step)


def test_moving_dual_step_equals_shifted_static():
    sc = moving_scene()
    assert np.abs(sc.obs_step).max() > 1.0  # really moving (metres per step)
    o = oracle.Oracle(sc)
    o.admm_iterate(3)
    s, zeta, xi, y0 = o.s.copy(), o.zeta.copy(), o.xi.copy(), o.y.copy()
    o.dual_sweep()
    for p in range(sc.n_pairs):
        b, t, A, bb, Cm, dv = shifted(sc, p)
        R, rho = oracle.pose(sc.pose_model, sc.pose_idx, sc.dim, s[b, t])
        y, st, piv, _ = oracle.pair_solve(A, bb, Cm, dv, R, rho, zeta[p], xi[p])
        assert st == o.status[p]
        if st == 0:
            n = len(y)
            np.testing.assert_allclose(o.y[p, :n], y, rtol=1e-9, atol=1e-11)


def test_moving_multiplier_equals_shifted_static():
    sc = moving_scene()
    o = oracle.Oracle(sc)
    o.admm_iterate(2)
    o.dual_sweep()
    o.primal_step()
    s, y, zeta0 = o.s.copy(), o.y.copy(), o.zeta.copy()
    o.multiplier_update()
    for p in range(sc.n_pairs):
        b, t, A, bb, Cm, dv = shifted(sc, p)
        R, rho = oracle.pose(sc.pose_model, sc.pose_idx, sc.dim, s[b, t])
        nr, no = A.shape[0], Cm.shape[0]
        mu, gam = y[p, nr:nr + no], y[p, nr + no]
        T = 1.0 + (dv - Cm @ rho) @ mu + gam  # Eq. 10 with d_j(t)
        assert abs((o.zeta[p] - zeta0[p]) - T) <= 1e-9 * (1.0 + abs(T))


def test_moving_scale_equals_shifted_static():
    sc = moving_scene()
    o = oracle.Oracle(sc)
    o.admm_iterate(2)
    alpha = o.scale_detect()
    for p in range(sc.n_pairs):
        b, t, A, bb, Cm, dv = shifted(sc, p)
        R, rho = oracle.pose(sc.pose_model, sc.pose_idx, sc.dim, o.s[b, t])
        a_ref, _ = oracle.scale_lp(A, bb, R, rho, Cm, dv)
        assert abs(alpha[p] - a_ref) <= 1e-9 * max(1.0, a_ref)


def test_zero_steps_equal_static_bitwise():
    sc = moving_scene()
    st = dataclasses.replace(sc, obs_step=np.zeros_like(sc.obs_step))
    still = dataclasses.replace(sc, obs_step=None)
    a, b = oracle.Oracle(st), oracle.Oracle(still)
    a.admm_iterate(3)
    b.admm_iterate(3)
    assert np.array_equal(a.s, b.s) and np.array_equal(a.y, b.y)
