"""Pins of the oracle's box block (state / control bounds of Eq. 13c-d, P:253-254,
inside IC_0 of P:289-290; NEXT f1; reading #7).

The oracle handles the boxes with one more ADMM block (consensus x = w, w in the
box, scaled multiplier l).  What pins it, independently of the oracle's code:

* zero obstacles, control bounds only: the converged iterate equals the optimum of
  the box-constrained LQ, condensed onto the controls and solved by scipy's bounded
  least squares (lsq_linear);
* zero obstacles, state and control bounds: the converged iterate satisfies the KKT
  conditions of the box-constrained LQ -- the active set read off the
  iterate, the equality-constrained QP on it solved densely (numpy), every bound
  multiplier of the right sign and the solution inside the box;
* bounds given but all infinite: bitwise the unbounded problem;
* one primal step: w = Pi_box(x + l_old), l_new - l_old = x - w, and the box term
  added to r_pri is sum ||x - w||^2.
"""
import dataclasses

import numpy as np
import pytest
from scipy.optimize import lsq_linear

import scenes
from test_oracle_admm import dense_kkt_lq, dyn, strip_obstacles

INF = np.inf


def lq_blocks(sc, b=0):
    """Dense data of the LQ of P:243-252: min 1/2 x^T H x + g^T x s.t. E x = e,
    x = (s_1..s_N, u_0..u_{N-1})."""
    N, ns, nu = sc.horizon, sc.n_state, sc.n_ctrl
    nx = N * ns + N * nu
    H, g = np.zeros((nx, nx)), np.zeros(nx)
    for t in range(1, N + 1):
        sl = slice((t - 1) * ns, t * ns)
        H[sl, sl] = 2 * sc.Qs
        g[sl] = -2 * sc.Qs @ sc.s_ref[b, t]
    for t in range(N):
        sl = slice(N * ns + t * nu, N * ns + (t + 1) * nu)
        H[sl, sl] = 2 * sc.Qu
    E, e = np.zeros((N * ns, nx)), np.zeros(N * ns)
    for t in range(N):
        A, B, c = dyn(sc, b, t)
        r = slice(t * ns, (t + 1) * ns)
        E[r, t * ns:(t + 1) * ns] = np.eye(ns)
        if t > 0:
            E[r, (t - 1) * ns:t * ns] = -A
        E[r, N * ns + t * nu:N * ns + (t + 1) * nu] = -B
        e[r] = c + (A @ sc.s0[b] if t == 0 else 0)
    return H, g, E, e


def box_vectors(sc):
    N, ns, nu = sc.horizon, sc.n_state, sc.n_ctrl
    f = lambda v, n, fill: np.full(n, fill) if v is None else np.asarray(v, float)
    lo = np.r_[np.tile(f(sc.s_min, ns, -INF), N), np.tile(f(sc.u_min, nu, -INF), N)]
    hi = np.r_[np.tile(f(sc.s_max, ns, INF), N), np.tile(f(sc.u_max, nu, INF), N)]
    return lo, hi


def aggressive_car(bounds_state: bool):
    """Zero-obstacle C2 car asked to jump 1.5 m sideways and back and speed up to 4 m/s:
    the unconstrained LQ optimum violates the boxes below."""
    sc = strip_obstacles(scenes.make_config(2))
    N = 20
    ref = sc.s_ref[:, :N + 1].copy()
    ref[:, 1:11, 1] = 1.5
    ref[:, 1:, 3] = 4.0
    kw = dict(u_min=np.array([-0.6, -0.4]), u_max=np.array([0.6, 0.4]), box_rho=2.0)
    if bounds_state:
        kw.update(s_min=np.array([-INF, -INF, -0.15, 2.0]), s_max=np.array([INF, 1.0, 0.15, 3.15]))
    return dataclasses.replace(sc, horizon=N, s_ref=ref, dyn_A=sc.dyn_A[:N], dyn_B=sc.dyn_B[:N],
                               dyn_c=sc.dyn_c[:N], **kw)


def quad_box():
    """Zero-obstacle C3 quadrotor (n_u = 4) with control bounds only."""
    sc = strip_obstacles(scenes.make_config(3))
    s_ref = sc.s_ref.copy()
    s_ref[:, 1:, 2] += 1.0  # climb a metre
    return dataclasses.replace(sc, s_ref=s_ref, u_min=np.full(sc.n_ctrl, -0.5), u_max=np.full(sc.n_ctrl, 0.5),
                               box_rho=5.0)


def xvec(o, b=0):
    return np.r_[o.s[b, 1:].reshape(-1), o.u[b].reshape(-1)]


@pytest.mark.parametrize("make", [lambda: aggressive_car(False), quad_box], ids=["car", "quad"])
def test_control_box_equals_bounded_least_squares(orc, make):
    sc = make()
    H, g, E, e = lq_blocks(sc)
    lo, hi = box_vectors(sc)
    N, ns, nu = sc.horizon, sc.n_state, sc.n_ctrl
    # condense x_s = F u + f0 (E_s x_s + E_u u = e with E_s invertible)
    Es, Eu = E[:, :N * ns], E[:, N * ns:]
    F = -np.linalg.solve(Es, Eu)
    f0 = np.linalg.solve(Es, e)
    Hs, Hu = H[:N * ns, :N * ns], H[N * ns:, N * ns:]
    Hc = F.T @ Hs @ F + Hu
    gc = F.T @ (Hs @ f0 + g[:N * ns])
    L = np.linalg.cholesky(Hc)  # 1/2 u^T Hc u + gc^T u = 1/2 ||L^T u + L^{-1} gc||^2 + const
    res = lsq_linear(L.T, -np.linalg.solve(L, gc), bounds=(lo[N * ns:], hi[N * ns:]), method="bvls",
                     tol=1e-14)
    u_ref = res.x
    unc = dense_kkt_lq(sc)[1].reshape(-1)
    assert np.any(unc > hi[N * ns:] + 0.05) or np.any(unc < lo[N * ns:] - 0.05)  # the box binds
    o = orc.Oracle(sc)
    hp, _, _ = o.admm_iterate(3000)
    np.testing.assert_allclose(o.u[0].reshape(-1), u_ref, atol=2e-7)
    assert hp[-1, 0] < 1e-12


def test_state_and_control_box_kkt_certificate(orc):
    sc = aggressive_car(True)
    o = orc.Oracle(sc)
    o.admm_iterate(4000)
    H, g, E, e = lq_blocks(sc)
    lo, hi = box_vectors(sc)
    x = xvec(o)
    at_lo = np.abs(x - lo) < 1e-6
    at_hi = np.abs(x - hi) < 1e-6
    act = np.flatnonzero(at_lo | at_hi)
    ns_x = sc.horizon * sc.n_state
    assert at_lo.any() and at_hi.any() and act.size >= 10
    assert (at_lo | at_hi)[:ns_x].sum() >= 3  # state bounds bind too
    # equality-constrained QP with the active bounds fixed: [H E^T I_A^T; E 0 0; I_A 0 0]
    nx, ne, na = len(x), E.shape[0], act.size
    IA = np.zeros((na, nx))
    IA[np.arange(na), act] = 1.0
    K = np.block([[H, E.T, IA.T], [E, np.zeros((ne, ne + na))], [IA, np.zeros((na, ne + na))]])
    rhs = np.r_[-g, e, np.where(at_lo[act], lo[act], hi[act])]
    sol = np.linalg.solve(K, rhs)
    xs, nu_a = sol[:nx], sol[nx + ne:]
    # H x + g + E^T pi + I_A^T nu = 0 with nu = -nu_lo (lower) or +nu_hi (upper), nu_lo, nu_hi >= 0
    assert np.all(nu_a[at_lo[act]] <= 1e-8) and np.all(nu_a[at_hi[act]] >= -1e-8)
    assert np.abs(nu_a).max() > 1e-3  # the box really binds
    assert np.all(xs >= lo - 1e-9) and np.all(xs <= hi + 1e-9)
    np.testing.assert_allclose(x, xs, atol=1e-6)


def test_infinite_bounds_equal_no_bounds_bitwise(orc):
    sc = scenes.make_config(2)
    inf_box = dataclasses.replace(sc, s_min=np.full(4, -INF), s_max=np.full(4, INF), u_min=np.full(2, -INF),
                                  u_max=np.full(2, INF), box_rho=7.0)
    a, b = orc.Oracle(sc), orc.Oracle(inf_box)
    ha = a.admm_iterate(5)
    hb = b.admm_iterate(5)
    assert np.array_equal(a.s, b.s) and np.array_equal(a.u, b.u) and np.array_equal(a.y, b.y)
    assert np.array_equal(ha[0], hb[0]) and np.array_equal(ha[1], hb[1])


def test_box_update_step(orc):
    sc = scenes.make_config(8)
    o = orc.Oracle(sc)
    o.admm_iterate(5)
    ws0, ls0, wu0, lu0 = o.ws.copy(), o.ls.copy(), o.wu.copy(), o.lu.copy()
    o.dual_sweep()
    o.primal_step()
    lo_s = np.where(np.isfinite(sc.s_min), sc.s_min, -INF)
    bs = np.isfinite(sc.s_min) | np.isfinite(sc.s_max)
    bu = np.isfinite(sc.u_min) | np.isfinite(sc.u_max)
    xs, xu = o.s[:, 1:], o.u
    ws = np.clip(xs + ls0[:, 1:], lo_s, sc.s_max)
    wu = np.clip(xu + lu0, sc.u_min, sc.u_max)
    np.testing.assert_array_equal(o.ws[:, 1:][..., bs], ws[..., bs])
    np.testing.assert_array_equal(o.wu[..., bu], wu[..., bu])
    np.testing.assert_allclose(o.ls[:, 1:][..., bs], (ls0[:, 1:] + xs - ws)[..., bs], atol=1e-14)
    np.testing.assert_allclose(o.lu[..., bu], (lu0 + xu - wu)[..., bu], atol=1e-14)
    r = ((xs - ws)[..., bs] ** 2).sum() + ((xu - wu)[..., bu] ** 2).sum()
    assert abs(o.boxres[0] - r) <= 1e-12 * (1 + r)
    rp_pairs = o.multiplier_update()
    assert o.boxres[0] > 0  # some bound was violated by the unprojected step


def test_c2b_converges_inside_the_box(orc):
    sc = scenes.make_config(8)
    o = orc.Oracle(sc)
    hp, hd, fails = o.admm_iterate(400)
    assert fails == 0 and hp[-1, 0] < 1e-6
    tol = 1e-3
    assert np.all(o.u >= sc.u_min - tol) and np.all(o.u <= sc.u_max + tol)
    assert np.all(o.s[:, 1:] >= sc.s_min - tol) and np.all(o.s[:, 1:] <= sc.s_max + tol)
    assert (np.abs(np.abs(o.wu) - sc.u_max) < 1e-9).sum() >= 3  # bounds bind
    assert o.scale_detect().min() > 0.99  # still (nearly) collision-free
