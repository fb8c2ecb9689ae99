"""Pins of the oracle's scale-based detection LP (Eq. 3) against
things other than itself: SPEC worked examples, the closed form for axis-aligned
boxes, scipy HiGHS on the primal LP and on the dual LP (Eq. 5, strong duality
P:152-155), the separating-axis theorem (alpha* > 1 iff disjoint) and
metamorphic scalings."""
import os

import numpy as np
import pytest
from scipy.optimize import linprog

from conftest import poly_from_vertices, random_convex_polygon, rot2, sat_disjoint_2d

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "spec_examples.txt")


def golden(kind):
    rows = []
    for line in open(GOLDEN):
        line = line.strip()
        if not line or line.startswith("#"):
            continue
        parts = [p.strip() for p in line.split("|")]
        if parts[0] == kind:
            rows.append([np.array([float(x) for x in p.split()]) for p in parts[1:]])
    assert rows, kind
    return rows


def box(center, half):
    d = len(center)
    A = np.zeros((2 * d, d))
    for k in range(d):
        A[2 * k, k], A[2 * k + 1, k] = 1.0, -1.0
    return A, np.repeat(np.asarray(half, float), 2) + A @ np.asarray(center, float)


def test_spec_examples(orc):
    Ar, br = box([0, 0], [1, 1])
    for inp, exp in golden("min_scale"):
        lo_x, hi_x, lo_y, hi_y = inp
        Co, do = box([(lo_x + hi_x) / 2, (lo_y + hi_y) / 2], [(hi_x - lo_x) / 2, (hi_y - lo_y) / 2])
        a, _ = orc.scale_lp(Ar, br, np.eye(2), np.zeros(2), Co, do)
        assert abs(a - exp[0]) < 1e-12, (inp, a, exp)


@pytest.mark.parametrize("d", [2, 3])
def test_box_closed_form(orc, d):
    rng = np.random.default_rng(10 + d)
    for _ in range(300):
        h = rng.uniform(0.2, 2.0, d)
        rho = rng.uniform(-3, 3, d)
        lo = rng.uniform(-4, 3, d)
        hi = lo + rng.uniform(0.1, 3.0, d)
        Ar, br = box(np.zeros(d), h)
        Co, do = box((lo + hi) / 2, (hi - lo) / 2)
        a, _ = orc.scale_lp(Ar, br, np.eye(d), rho, Co, do)
        closed = max(0.0, np.max(np.maximum(lo - rho, rho - hi) / h))
        assert abs(a - closed) <= 1e-9 * max(1.0, closed), (a, closed)


def highs_primal(A, b, R, rho, Co, do):
    d = A.shape[1]
    G1 = np.hstack([A @ R.T, -b[:, None]])
    h1 = A @ R.T @ rho
    G2 = np.hstack([Co, np.zeros((Co.shape[0], 1))])
    res = linprog(np.r_[np.zeros(d), 1.0], A_ub=np.vstack([G1, G2]), b_ub=np.r_[h1, do],
                  bounds=[(None, None)] * (d + 1), method="highs")
    assert res.status == 0
    return res.fun


def highs_dual(A, b, R, rho, Co, do):
    """Eq. 5 for the posed pair: max -(d - C rho)^T mu, b^T lam = 1, A^T lam + (C R)^T mu = 0."""
    nr, no, d = A.shape[0], Co.shape[0], A.shape[1]
    Aeq = np.zeros((1 + d, nr + no))
    Aeq[0, :nr] = b
    Aeq[1:, :nr] = A.T
    Aeq[1:, nr:] = (Co @ R).T
    res = linprog(np.r_[np.zeros(nr), do - Co @ rho], A_eq=Aeq, b_eq=np.r_[1.0, np.zeros(d)],
                  bounds=[(0, None)] * (nr + no), method="highs")
    assert res.status == 0
    return -res.fun, res.x


def test_vs_highs_primal_and_dual_2d(orc):
    rng = np.random.default_rng(7)
    for _ in range(200):
        Vr = random_convex_polygon(rng, [0.0, 0.0], 0.5, 2.0)
        Ar, br = poly_from_vertices(Vr)
        Vo = random_convex_polygon(rng, rng.uniform(-4, 4, 2), 0.3, 2.5)
        Co, do = poly_from_vertices(Vo)
        R, rho = rot2(rng.uniform(-np.pi, np.pi)), rng.uniform(-2, 2, 2)
        a, _ = orc.scale_lp(Ar, br, R, rho, Co, do)
        ap = highs_primal(Ar, br, R, rho, Co, do)
        ad, _ = highs_dual(Ar, br, R, rho, Co, do)
        assert abs(a - ap) <= 1e-7 * max(1, ap)
        assert abs(a - ad) <= 1e-7 * max(1, ad)


def test_vs_highs_3d_rotated_boxes(orc):
    rng = np.random.default_rng(8)
    for _ in range(100):
        Ar, br = box(np.zeros(3), rng.uniform(0.1, 1.0, 3))
        Q, _ = np.linalg.qr(rng.standard_normal((3, 3)))
        Co, do = box(np.zeros(3), rng.uniform(0.2, 1.5, 3))
        c = rng.uniform(-3, 3, 3)
        Co = Co @ Q.T
        do = do + Co @ c
        psi = rng.uniform(-np.pi, np.pi)
        R = np.eye(3)
        R[:2, :2] = rot2(psi)
        rho = rng.uniform(-1, 1, 3)
        a, _ = orc.scale_lp(Ar, br, R, rho, Co, do)
        ap = highs_primal(Ar, br, R, rho, Co, do)
        assert abs(a - ap) <= 1e-7 * max(1, ap)


def test_alpha_gt_one_iff_disjoint_sat(orc):
    rng = np.random.default_rng(9)
    n_dis = n_int = 0
    for _ in range(400):
        Vr = random_convex_polygon(rng, [0.0, 0.0], 0.5, 1.5)
        Ar, br = poly_from_vertices(Vr)
        Vo = random_convex_polygon(rng, rng.uniform(-3, 3, 2), 0.3, 1.5)
        Co, do = poly_from_vertices(Vo)
        th, rho = rng.uniform(-np.pi, np.pi), rng.uniform(-1, 1, 2)
        R = rot2(th)
        a, _ = orc.scale_lp(Ar, br, R, rho, Co, do)
        if abs(a - 1.0) <= 1e-6:
            continue
        posed = Vr @ R.T + rho
        dis = sat_disjoint_2d(posed, Vo)
        assert (a > 1.0) == dis, (a, dis)
        n_dis += dis
        n_int += not dis
    assert n_dis > 50 and n_int > 50


def test_metamorphic(orc):
    rng = np.random.default_rng(11)
    for _ in range(100):
        Ar, br = poly_from_vertices(random_convex_polygon(rng, [0, 0], 0.5, 1.5))
        Co, do = poly_from_vertices(random_convex_polygon(rng, rng.uniform(-3, 3, 2), 0.3, 1.5))
        R, rho = rot2(rng.uniform(-3, 3)), rng.uniform(-1, 1, 2)
        a, _ = orc.scale_lp(Ar, br, R, rho, Co, do)
        s = rng.uniform(0.3, 3.0)  # robot scaled by s => alpha*/s
        a2, _ = orc.scale_lp(Ar, s * br, R, rho, Co, do)
        assert abs(a2 - a / s) <= 1e-9 * max(1, a)
        w1, w2 = rng.uniform(0.2, 5, len(br)), rng.uniform(0.2, 5, len(do))  # positive row scaling
        a3, _ = orc.scale_lp(Ar * w1[:, None], br * w1, R, rho, Co * w2[:, None], do * w2)
        assert abs(a3 - a) <= 1e-9 * max(1, a)
        Q, t = rot2(rng.uniform(-3, 3)), rng.uniform(-5, 5, 2)  # joint rigid motion
        a4, _ = orc.scale_lp(Ar, br, Q @ R, Q @ rho + t, Co @ Q.T, do + (Co @ Q.T) @ t)
        assert abs(a4 - a) <= 1e-9 * max(1, a)
