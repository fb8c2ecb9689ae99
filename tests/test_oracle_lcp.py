"""Pins of the oracle's per-pair QP (Eq. 19), its equality
elimination, QP->LCP conversion and Lemke:
SPEC worked examples, brute-force 2^n complementary-basis enumeration, the KKT
certificate of Eq. 19, scipy SLSQP on Eq. 19, the slab closed form, the
strong-duality link optimum == 0 <=> alpha* >= 1, sigma invariance."""
import itertools
import os

import numpy as np
import pytest
from scipy.optimize import minimize

from conftest import poly_from_vertices, random_convex_polygon, rot2
from test_oracle_scale import golden, highs_dual


def random_pair(rng, sep=None, nmax_o=6):
    """Robot polygon containing its origin; obstacle polygon near it; random pose."""
    Ar, br = poly_from_vertices(random_convex_polygon(rng, [0, 0], 0.6, 1.5, 3, 4))
    c = rng.uniform(-2.5, 2.5, 2)
    Co, do = poly_from_vertices(random_convex_polygon(rng, c, 0.4, 1.5, 3, nmax_o))
    R, rho = rot2(rng.uniform(-np.pi, np.pi)), rng.uniform(-0.5, 0.5, 2)
    return Ar, br, Co, do, R, rho


def qp_objective(K, bvec, y):
    u = K.T @ y + bvec
    return 0.5 * u @ u


def test_spec_lemke_examples(orc):
    for n, M, q, z in golden("lemke"):
        n = int(n[0])
        zz, st, piv, _ = orc.lemke(M.reshape(n, n), q)
        assert st == 0
        np.testing.assert_allclose(zz, z, atol=1e-14)


def enumerate_lcp(M, q, tol=1e-9):
    """All complementary-basis solutions of w = Mz + q, w,z >= 0, w^T z = 0 (n <= 12)."""
    n = len(q)
    sols = []
    for mask in itertools.product([0, 1], repeat=n):
        S = [i for i in range(n) if mask[i]]
        z = np.zeros(n)
        if S:
            Mss = M[np.ix_(S, S)]
            if abs(np.linalg.det(Mss)) < 1e-12:
                continue
            z[S] = np.linalg.solve(Mss, -q[S])
        w = M @ z + q
        sc = 1 + np.abs(q).max()
        if z.min() >= -tol * sc and w.min() >= -tol * sc:
            sols.append(z)
    return sols


def lcp_valid(M, q, z, tol=1e-9):
    w = M @ z + q
    sc = 1 + np.abs(q).max()
    return z.min() >= -tol * sc and w.min() >= -tol * sc and abs(w @ z) <= tol * sc * (1 + np.abs(z).max())


def test_lemke_vs_enumeration(orc):
    rng = np.random.default_rng(21)
    n_unique = 0
    for trial in range(120):
        Ar, br, Co, do, R, rho = random_pair(rng, nmax_o=5)
        zeta, xi = rng.normal(0, 0.3), rng.normal(0, 0.3, 2)
        K, bvec, e, M, q = orc.pair_lcp(Ar, br, Co, do, R, rho, zeta, xi)
        if len(q) > 10:
            continue
        z, st, piv, _ = orc.lemke(M, q)
        assert st == 0
        assert lcp_valid(M, q, z)
        sols = enumerate_lcp(M, q)
        assert sols, "enumeration found no solution"
        # y_U part (all but phi) unique among enumerated solutions => Lemke must match it
        Y = np.array([s[:-1] for s in sols])
        if np.ptp(Y, axis=0).max() < 1e-9:
            n_unique += 1
            np.testing.assert_allclose(z[:-1], Y[0], atol=1e-9)
        else:
            # non-unique y_U: every LCP solution is a QP optimum (convex), so Lemke's choice
            # must reach the same reduced objective as every enumerated solution
            def f(v):
                return 0.5 * v @ M[:-1, :-1] @ v + q[:-1] @ v
            fs = [f(s) for s in Y]
            assert abs(f(z[:-1]) - min(fs)) <= 1e-9 * (1 + abs(min(fs)))
            assert np.ptp(fs) <= 1e-8 * (1 + abs(min(fs)))
    assert n_unique > 10


def kkt_check(K, bvec, kappa, y, tol=1e-9):
    """Eq. 19 KKT: g = K(K^T y + b); exists nu: g - nu kappa >= 0, = 0 on supp(y)."""
    g = K @ (K.T @ y + bvec)
    lam = kappa > 0
    nu = np.min(g[lam] / kappa[lam])
    r = g - nu * kappa
    sc = 1 + np.abs(g).max()
    assert r.min() >= -tol * sc
    assert np.all(np.abs(r[y > 1e-9]) <= tol * sc * 10)
    assert abs(kappa @ y - 1) <= 1e-12
    assert y.min() >= -1e-12


def test_pair_qp_kkt_and_slsqp(orc):
    rng = np.random.default_rng(22)
    for trial in range(150):
        Ar, br, Co, do, R, rho = random_pair(rng)
        zeta, xi = rng.normal(0, 0.5), rng.normal(0, 0.5, 2)
        y, st, piv, _ = orc.pair_solve(Ar, br, Co, do, R, rho, zeta, xi)
        assert st == 0
        K, bvec, e, M, q = orc.pair_lcp(Ar, br, Co, do, R, rho, zeta, xi)
        kappa = np.r_[br, np.zeros(len(do) + 1)]
        kkt_check(K, bvec, kappa, y)
        # independent solver on Eq. 19 directly
        n = len(y)
        y0 = np.r_[np.ones(len(br)) / br.sum(), np.zeros(n - len(br))]
        res = minimize(lambda v: qp_objective(K, bvec, v), y0, jac=lambda v: K @ (K.T @ v + bvec),
                       bounds=[(0, None)] * n, constraints=[{"type": "eq", "fun": lambda v: kappa @ v - 1,
                                                              "jac": lambda v: kappa}],
                       method="SLSQP", options={"ftol": 1e-14, "maxiter": 2000})
        fo, fs = qp_objective(K, bvec, y), res.fun
        assert fo <= fs + 1e-9 * (1 + fs)
        assert fs - fo <= 1e-6 * (1 + fo)
        # the residual vector u* = K^T y + b is unique (strict convexity in u)
        us, uo = K.T @ res.x + bvec, K.T @ y + bvec
        assert np.abs(us - uo).max() <= 2e-4 * (1 + np.abs(uo).max())


def test_elimination_round_trip(orc):
    """Eqs. 20-21: y_e recovered from y_U gives kappa^T y = eta; reduced objective == full."""
    rng = np.random.default_rng(23)
    for trial in range(100):
        Ar, br, Co, do, R, rho = random_pair(rng)
        zeta, xi = rng.normal(0, 0.5), rng.normal(0, 0.5, 2)
        K, bvec, e, M, q = orc.pair_lcp(Ar, br, Co, do, R, rho, zeta, xi)
        assert e == int(np.argmax(br))
        n = K.shape[0]
        U = [k for k in range(n) if k != e]
        kap = np.r_[br, np.zeros(n - len(br))]
        yU = rng.uniform(0, 1, n - 1)
        ye = (1 - kap[U] @ yU) / kap[e]
        y = np.zeros(n)
        y[U], y[e] = yU, ye
        assert abs(kap @ y - 1) < 1e-12
        # reduced QP objective via the LCP data: 1/2 ||Kt^T yU + bt||^2 where M_UU = Kt Kt^T,
        # q_U = Kt bt  =>  f = 1/2 yU^T M_UU yU + q_U^T yU + 1/2 ||bt||^2
        Kt = K[U] - np.outer(kap[U] / kap[e], K[e])
        bt = bvec + K[e] / kap[e]
        np.testing.assert_allclose(M[:-1, :-1], Kt @ Kt.T, rtol=1e-13, atol=1e-13)
        np.testing.assert_allclose(q[:-1], Kt @ bt, rtol=1e-13, atol=1e-12)
        f_red = 0.5 * yU @ M[:-1, :-1] @ yU + q[:-1] @ yU + 0.5 * bt @ bt
        assert abs(f_red - qp_objective(K, bvec, y)) <= 1e-10 * (1 + f_red)
        assert q[-1] == 1.0 / kap[e]
        np.testing.assert_allclose(M[:-1, -1], kap[U] / kap[e])
        np.testing.assert_allclose(M[-1, :-1], -kap[U] / kap[e])


def test_slab_closed_form(orc):
    """Robot box (half-length h along x, half-width w) at the origin, obstacle box whose
    near face x = g < h faces it and whose lateral extent covers the robot origin,
    zeta = xi = 0: f* = 1/2 (1-a)^2/(1+g^2), u* = (1-a)/(1+g^2) (1,-g,0), a = g/h."""
    for h, w, g in [(1.0, 0.5, 0.3), (2.25, 1.0, 1.1), (1.5, 1.5, 0.05), (0.8, 0.4, 0.7), (2.0, 0.3, 1.9)]:
        Ar = np.array([[1.0, 0], [-1, 0], [0, 1], [0, -1]])
        br = np.array([h, h, w, w])
        Co = Ar.copy()
        do = np.array([g + 3.0, -g, 4.0, 4.0])  # x in [g, g+3], |y| <= 4
        y, st, piv, _ = orc.pair_solve(Ar, br, Co, do, np.eye(2), np.zeros(2), 0.0, np.zeros(2))
        K, bvec, e, M, q = orc.pair_lcp(Ar, br, Co, do, np.eye(2), np.zeros(2), 0.0, np.zeros(2))
        a = g / h
        u = K.T @ y + bvec
        np.testing.assert_allclose(u, (1 - a) / (1 + g * g) * np.array([1.0, -g, 0.0]), atol=1e-12)
        assert abs(qp_objective(K, bvec, y) - 0.5 * (1 - a) ** 2 / (1 + g * g)) < 1e-13


def test_optimum_zero_iff_separated(orc):
    """At zeta = xi = 0 the pair-QP optimum is 0 iff the dual LP (Eq. 5) reaches >= 1,
    i.e. iff alpha* >= 1."""
    rng = np.random.default_rng(24)
    seen = [0, 0]
    for trial in range(200):
        Ar, br, Co, do, R, rho = random_pair(rng)
        a, _ = orc.scale_lp(Ar, br, R, rho, Co, do)
        ad, _ = highs_dual(Ar, br, R, rho, Co, do)
        if abs(ad - 1) < 1e-6:
            continue
        y, st, piv, _ = orc.pair_solve(Ar, br, Co, do, R, rho, 0.0, np.zeros(2))
        K, bvec, *_ = orc.pair_lcp(Ar, br, Co, do, R, rho, 0.0, np.zeros(2))
        f = qp_objective(K, bvec, y)
        assert (f <= 1e-20) == (ad > 1), (f, ad, a)
        seen[ad > 1] += 1
    assert min(seen) > 30


def test_lemke_scale_equivariance(orc):
    rng = np.random.default_rng(25)
    for trial in range(50):
        Ar, br, Co, do, R, rho = random_pair(rng)
        K, bvec, e, M, q = orc.pair_lcp(Ar, br, Co, do, R, rho, rng.normal(), rng.normal(0, 1, 2))
        z1, *_ = orc.lemke(M, q)
        c = 4.0  # power of two: exact scaling of every tableau entry
        z2, *_ = orc.lemke(M, c * q)
        np.testing.assert_allclose(z2, c * z1, rtol=1e-12, atol=1e-14)


def test_sigma_invariance_of_dual_step(orc):
    """Eq. 15's argmin does not depend on sigma (P:356 'equivalent'): bitwise."""
    import scenes

    sc = scenes.make_config(2)
    ys = []
    for sigma in (1.0, 300.0, 1e4):
        o = orc.Oracle(sc, sigma=sigma)
        o.zeta[:] = np.linspace(-0.3, 0.3, len(o.zeta))
        o.dual_sweep()
        ys.append(o.y.copy())
    assert np.array_equal(ys[0], ys[1]) and np.array_equal(ys[1], ys[2])


def test_prox_zero_is_paper_exact(orc):
    rng = np.random.default_rng(26)
    Ar, br, Co, do, R, rho = random_pair(rng)
    a = orc.pair_lcp(Ar, br, Co, do, R, rho, 0.1, np.array([0.2, -0.1]))
    b = orc.pair_lcp(Ar, br, Co, do, R, rho, 0.1, np.array([0.2, -0.1]), prox_eps=0.0,
                     y_prev=rng.uniform(0, 1, len(br) + len(do) + 1))
    assert np.array_equal(a[3], b[3]) and np.array_equal(a[4], b[4])


def test_prox_unique_minimiser_kkt(orc):
    """prox_eps > 0 (reading #2): y minimises Eq. 19a + eps/2 ||y - y_prev||^2 (KKT)."""
    rng = np.random.default_rng(27)
    eps = 1e-3
    for trial in range(50):
        Ar, br, Co, do, R, rho = random_pair(rng)
        n = len(br) + len(do) + 1
        yp = rng.uniform(0, 0.5, n)
        zeta, xi = rng.normal(0, 0.5), rng.normal(0, 0.5, 2)
        y, st, *_ = orc.pair_solve(Ar, br, Co, do, R, rho, zeta, xi, prox_eps=eps, y_prev=yp)
        K, bvec, *_ = orc.pair_lcp(Ar, br, Co, do, R, rho, zeta, xi)
        kappa = np.r_[br, np.zeros(len(do) + 1)]
        g = K @ (K.T @ y + bvec) + eps * (y - yp)
        lam = kappa > 0
        nu = np.min(g[lam] / kappa[lam])
        r = g - nu * kappa
        assert r.min() >= -1e-9 * (1 + np.abs(g).max())
        assert np.all(np.abs(r[y > 1e-9]) <= 1e-8 * (1 + np.abs(g).max()))
