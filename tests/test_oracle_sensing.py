"""Pins of the oracle's sensing filter ("can only sense the obstacles within
20m x 20m x 6m"): obstacle (b, j) enters the (i, j, t) table
iff it meets the world-aligned box rho(s0_b) + [-h, h].

* orc_sense agrees with an independent LP feasibility test (scipy HiGHS: the largest
  common slack of the obstacle's and the box's inequalities), away from touching;
* a filtered problem IS the problem with the unsensed obstacles removed: the same
  trajectory and the same certificates for the sensed pairs after K iterations;
* unsensed pairs keep their cold-start certificates and report alpha = +inf.
"""
import dataclasses

import numpy as np
import pytest
from scipy.optimize import linprog

import scenes


def lp_slack(Cm, dv, centre, half):
    """max t s.t. C y + t <= d, (y - centre) <= h - t, -(y - centre) <= h - t."""
    d = Cm.shape[1]
    norms = np.r_[np.linalg.norm(Cm, axis=1), np.ones(2 * d)]
    A = np.r_[Cm, np.eye(d), -np.eye(d)]
    b = np.r_[dv, centre + half, half - centre]
    res = linprog(np.r_[np.zeros(d), -1.0], A_ub=np.c_[A, norms], b_ub=b, bounds=[(None, None)] * (d + 1),
                  method="highs")
    assert res.status == 0
    return -res.fun


def sensing_cases():
    c4 = dataclasses.replace(scenes.make_config(4), sense_half=np.array([30.0, 5.0]))
    c5 = dataclasses.replace(scenes.make_c5(scene_ids=[0, 7, 4000]), sense_half=np.array([25.0, 25.0]))
    c3 = dataclasses.replace(scenes.make_config(3), sense_half=np.array([4.0, 1.0, 0.6]))
    return [c4, c5, c3]


@pytest.mark.parametrize("k", range(3))
def test_sense_equals_lp_feasibility(orc, k):
    sc = sensing_cases()[k]
    o = orc.Oracle(sc)
    assert 0 < o.sensed.sum() < o.sensed.size  # the filter bites
    for b in range(sc.n_scenes):
        R, rho = orc.pose(sc.pose_model, sc.pose_idx, sc.dim, sc.s0[b])
        for j in range(sc.n_obs):
            lo, hi = sc.obs_off[b * sc.n_obs + j], sc.obs_off[b * sc.n_obs + j + 1]
            t = lp_slack(sc.obs_C[lo:hi], sc.obs_d[lo:hi], rho, sc.sense_half)
            if abs(t) > 1e-7:
                assert o.sensed[b * sc.n_obs + j] == (t > 0), (b, j, t)


def only_sensed(sc, sensed):
    keep = np.flatnonzero(sensed)
    offs, Cs, ds = [0], [], []
    for j in keep:
        lo, hi = sc.obs_off[j], sc.obs_off[j + 1]
        Cs.append(sc.obs_C[lo:hi])
        ds.append(sc.obs_d[lo:hi])
        offs.append(offs[-1] + hi - lo)
    step = None if sc.obs_step is None else np.ascontiguousarray(sc.obs_step[keep])
    return dataclasses.replace(sc, n_obs=len(keep), obs_off=np.asarray(offs, np.int32), obs_C=np.concatenate(Cs),
                               obs_d=np.concatenate(ds), obs_step=step, sense_half=None), keep


def test_filtered_problem_is_the_reduced_problem(orc):
    sc = scenes.make_config(9)
    o = orc.Oracle(sc)
    red, keep = only_sensed(sc, o.sensed)
    r = orc.Oracle(red)
    K = 40
    hp, hd, f = o.admm_iterate(K)
    hp2, hd2, f2 = r.admm_iterate(K)
    np.testing.assert_allclose(o.s, r.s, rtol=0, atol=1e-9)
    np.testing.assert_allclose(o.u, r.u, rtol=0, atol=1e-9)
    np.testing.assert_allclose(hp, hp2, rtol=1e-9, atol=1e-12)
    np.testing.assert_allclose(hd, hd2, rtol=1e-9, atol=1e-12)
    N, M, Mr = sc.horizon, sc.n_obs, red.n_obs
    y = o.y.reshape(N, sc.n_parts, M, -1)
    y2 = r.y.reshape(N, red.n_parts, Mr, -1)
    np.testing.assert_allclose(y[:, :, keep, :y2.shape[-1]], y2, atol=1e-8)
    # unsensed pairs: cold-start certificates, alpha = +inf
    o0 = orc.Oracle(sc)
    drop = np.setdiff1d(np.arange(M), keep)
    assert np.array_equal(y[:, :, drop], o0.y.reshape(N, sc.n_parts, M, -1)[:, :, drop])
    alpha = o.scale_detect().reshape(N, sc.n_parts, M)
    assert np.all(np.isinf(alpha[:, :, drop])) and np.all(np.isfinite(alpha[:, :, keep]))
    np.testing.assert_allclose(alpha[:, :, keep], r.scale_detect().reshape(N, red.n_parts, Mr), rtol=1e-12)
