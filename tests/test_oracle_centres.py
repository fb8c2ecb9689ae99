"""Pins of per-part scaling centres (reading #22): part i
is scaled about a body-frame point o_i inside it instead of the body origin.

* the scale factor alpha* (Eq. 3 about o_i) equals scipy HiGHS's LP optimum written
  from the definition (min alpha s.t. A_i (R^T (y - rho) - o_i) <= alpha b~_i,
  C_j y <= d_j), and alpha* <= 1 iff the part and obstacle intersect (an LP
  feasibility test that never mentions o_i);
* the GN primal step with centres == least squares on finite-difference-linearised
  residuals (test_oracle_admm.test_gn_primal_step_vs_fd_least_squares[10]);
* cold start lambda = 1 / sum(b~_i); centres at the origin == no centres, bitwise.
"""
import dataclasses

import numpy as np
from scipy.optimize import linprog

import scenes


def part_rows(sc, i):
    return sc.part_A[sc.part_off[i]:sc.part_off[i + 1]], sc.part_b[sc.part_off[i]:sc.part_off[i + 1]]


def test_scale_about_centre_equals_lp(orc):
    sc = scenes.make_config(10)
    o = orc.Oracle(sc)
    o.admm_iterate(20)
    alpha = o.scale_detect()
    N, npart, M, d = sc.horizon, sc.n_parts, sc.n_obs, sc.dim
    checked = 0
    for t in range(1, N + 1, 3):
        R, rho = orc.pose(sc.pose_model, sc.pose_idx, d, o.s[0, t])
        for i in range(npart):
            A, b = part_rows(sc, i)
            oc = sc.part_ctr[i]
            bt = b - A @ oc
            for j in range(M):
                Cm, dv = sc.obs_C[sc.obs_off[j]:sc.obs_off[j + 1]], sc.obs_d[sc.obs_off[j]:sc.obs_off[j + 1]]
                # variables (y, alpha): A R^T y - alpha b~ <= A R^T rho + A o_i, C y <= d
                G = np.r_[np.c_[A @ R.T, -bt], np.c_[Cm, np.zeros(len(dv))]]
                h = np.r_[A @ R.T @ rho + A @ oc, dv]
                res = linprog(np.r_[np.zeros(d), 1.0], A_ub=G, b_ub=h, bounds=[(None, None)] * (d + 1),
                              method="highs")
                p = ((t - 1) * npart + i) * M + j
                assert abs(alpha[p] - res.fun) <= 1e-8 * max(1.0, abs(res.fun))
                # classification without the centre: the part itself (A R^T (y - rho) <= b)
                feas = linprog(np.zeros(d), A_ub=np.r_[A @ R.T, Cm], b_ub=np.r_[b + A @ R.T @ rho, dv],
                               bounds=[(None, None)] * d, method="highs")
                if abs(alpha[p] - 1.0) > 1e-6:
                    assert (feas.status == 0) == (alpha[p] < 1.0)
                checked += 1
    assert checked > 50


def test_cold_start_uses_shifted_offsets(orc):
    sc = scenes.make_config(10)
    o = orc.Oracle(sc)
    for i in range(sc.n_parts):
        A, b = part_rows(sc, i)
        bt = b - A @ sc.part_ctr[i]
        assert np.all(bt > 0) and (i == 0 or np.any(b <= 0))  # the trailer needs its centre
        p = i * sc.n_obs
        np.testing.assert_allclose(o.y[p, :len(b)], 1.0 / bt.sum(), rtol=1e-15)


def test_centres_at_origin_equal_no_centres_bitwise(orc):
    sc = scenes.make_config(2)
    zc = dataclasses.replace(sc, part_ctr=np.zeros((sc.n_parts, sc.dim)))
    a, b = orc.Oracle(sc), orc.Oracle(zc)
    ha = a.admm_iterate(5)
    hb = b.admm_iterate(5)
    assert np.array_equal(a.s, b.s) and np.array_equal(a.y, b.y)
    assert np.array_equal(ha[0], hb[0])
    assert np.array_equal(a.scale_detect(), b.scale_detect())
