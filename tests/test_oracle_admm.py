"""Pins of the oracle's ADMM steps 2-3 (Eqs. 16-17) and of the
whole iteration: zero-obstacle step == dense-KKT LQ optimum,
the Gauss-Newton primal step == least squares on finite-difference-linearised
residuals, exact dynamics feasibility, multiplier update == 0 on LP-duality
certificates (P:152-163 with Eqs. 10-11), SPEC multiplier example, translation
equivariance and obstacle-permutation invariance of K iterations."""
import dataclasses

import numpy as np
import pytest
from scipy.optimize import linprog

import scenes
from test_oracle_scale import golden


def strip_obstacles(sc):
    return dataclasses.replace(sc, n_obs=0, obs_off=np.zeros(sc.n_scenes * 0 + 1, np.int32),
                               obs_C=np.zeros((0, sc.dim)), obs_d=np.zeros(0))


def dyn(sc, b, t):
    nt = sc.horizon if sc.dyn_per_time else 1
    i = (b * nt if sc.dyn_per_scene else 0) + (t if sc.dyn_per_time else 0)
    return sc.dyn_A[i], sc.dyn_B[i], sc.dyn_c[i]


def dense_kkt_lq(sc, b=0):
    """min sum_{t>=1} ||s_t - sref_t||^2_Qs + sum_{t<N} ||u_t||^2_Qu  s.t. dynamics."""
    N, ns, nu = sc.horizon, sc.n_state, sc.n_ctrl
    nx = N * ns + N * nu
    H = np.zeros((nx, nx))
    g = np.zeros(nx)
    for t in range(1, N + 1):
        sl = slice((t - 1) * ns, t * ns)
        H[sl, sl] = 2 * sc.Qs
        g[sl] = -2 * sc.Qs @ sc.s_ref[b, t]
    for t in range(N):
        sl = slice(N * ns + t * nu, N * ns + (t + 1) * nu)
        H[sl, sl] = 2 * sc.Qu
    E = np.zeros((N * ns, nx))
    e = np.zeros(N * ns)
    for t in range(N):
        A, B, c = dyn(sc, b, t)
        r = slice(t * ns, (t + 1) * ns)
        E[r, t * ns:(t + 1) * ns] = np.eye(ns)  # s_{t+1}
        if t > 0:
            E[r, (t - 1) * ns:t * ns] = -A
        E[r, N * ns + t * nu:N * ns + (t + 1) * nu] = -B
        e[r] = c + (A @ sc.s0[b] if t == 0 else 0)
    KKT = np.block([[H, E.T], [E, np.zeros((N * ns, N * ns))]])
    sol = np.linalg.solve(KKT, np.r_[-g, e])
    return sol[:N * ns].reshape(N, ns), sol[N * ns:nx].reshape(N, nu)


@pytest.mark.parametrize("cfg", [1, 2, 3, 11, 12])
def test_zero_obstacles_is_dense_lq(orc, cfg):
    sc = strip_obstacles(scenes.make_config(cfg))
    o = orc.Oracle(sc)
    o.admm_iterate(1)
    s, u = dense_kkt_lq(sc)
    np.testing.assert_allclose(o.s[0, 1:], s, rtol=1e-9, atol=1e-9)
    np.testing.assert_allclose(o.u[0], u, rtol=1e-9, atol=1e-9)
    s1, u1 = o.s.copy(), o.u.copy()
    o.admm_iterate(1)  # converged after one iteration
    np.testing.assert_allclose(o.s, s1, atol=1e-12)
    np.testing.assert_allclose(o.u, u1, atol=1e-12)


# ---------------------------------------------------------------------------
# Gauss-Newton primal step vs least squares on FD-linearised residuals
# ---------------------------------------------------------------------------

def pose_of(sc, st):
    d = sc.dim
    rho = st[sc.pose_idx[:d]]
    R = np.eye(d)
    if sc.pose_model != scenes.POSE_TRANSLATION:
        th = st[sc.pose_idx[d]]
        R[:2, :2] = [[np.cos(th), -np.sin(th)], [np.sin(th), np.cos(th)]]
    return R, rho


def pair_residual(sc, y, zeta, xi, b, t, i, j, st):
    """r_p(s_t) = (T_p + zeta, R_p + xi) from the geometric definitions."""
    d = sc.dim
    R, rho = pose_of(sc, st)
    if getattr(sc, "part_ctr", None) is not None:  # part scaled about its centre o_i (NEXT f3)
        rho = rho + R @ sc.part_ctr[i]
    A = sc.part_A[sc.part_off[i]:sc.part_off[i + 1]]
    o = b * sc.n_obs + j
    Cm = sc.obs_C[sc.obs_off[o]:sc.obs_off[o + 1]]
    dv = sc.obs_d[sc.obs_off[o]:sc.obs_off[o + 1]]
    nr, no = len(A), len(dv)
    lam, mu, gam = y[:nr], y[nr:nr + no], y[nr + no]
    T = 1 + (dv - Cm @ rho) @ mu + gam
    Rr = A.T @ lam + (Cm @ R).T @ mu
    return np.r_[T + zeta, Rr + xi]


@pytest.mark.parametrize("cfg", [2, 3, 10, 11, 12])
def test_gn_primal_step_vs_fd_least_squares(orc, cfg):
    sc = scenes.make_config(cfg)
    o = orc.Oracle(sc)
    o.admm_iterate(3)          # a non-trivial iterate
    o.dual_sweep()             # y^{k+1} at s^k
    sk, y, zeta, xi = o.s.copy(), o.y.copy(), o.zeta.copy(), o.xi.copy()
    o.primal_step()
    N, ns, nu, d = sc.horizon, sc.n_state, sc.n_ctrl, sc.dim
    npc = d if sc.pose_model == scenes.POSE_TRANSLATION else d + 1
    pidx = sc.pose_idx[:npc]
    # affine map U -> s_t (t = 1..N)
    m = N * nu
    F = np.zeros((ns, m))
    f = sc.s0[0].copy()
    Fs, fs = [], []
    for t in range(N):
        A, B, c = dyn(sc, 0, t)
        F = A @ F
        F[:, t * nu:(t + 1) * nu] += B
        f = A @ f + c
        Fs.append(F.copy())
        fs.append(f.copy())
    rows, rhs = [], []
    Ls, Lu = np.linalg.cholesky(sc.Qs).T, np.linalg.cholesky(sc.Qu).T
    for t in range(1, N + 1):
        rows.append(Ls @ Fs[t - 1])
        rhs.append(-Ls @ (fs[t - 1] - sc.s_ref[0, t]))
    for t in range(N):
        Sel = np.zeros((nu, m))
        Sel[:, t * nu:(t + 1) * nu] = np.eye(nu)
        rows.append(Lu @ Sel)
        rhs.append(np.zeros(nu))
    w = np.sqrt(sc.sigma / 2)
    h = 1e-6
    p = 0
    for t in range(1, N + 1):
        for i in range(sc.n_parts):
            for j in range(sc.n_obs):
                st = sk[0, t]
                r0 = pair_residual(sc, y[p], zeta[p], xi[p], 0, t, i, j, st)
                J = np.zeros((d + 1, npc))
                for a in range(npc):
                    e = np.zeros(ns)
                    e[pidx[a]] = h
                    J[:, a] = (pair_residual(sc, y[p], zeta[p], xi[p], 0, t, i, j, st + e)
                               - pair_residual(sc, y[p], zeta[p], xi[p], 0, t, i, j, st - e)) / (2 * h)
                P = np.zeros((npc, ns))
                P[np.arange(npc), pidx] = 1
                rows.append(w * J @ P @ Fs[t - 1])
                rhs.append(-w * (r0 + J @ P @ (fs[t - 1] - st)))
                p += 1
    U, *_ = np.linalg.lstsq(np.vstack(rows), np.concatenate(rhs), rcond=None)
    np.testing.assert_allclose(o.u[0].ravel(), U, rtol=1e-6, atol=1e-6)
    # dynamics hold exactly along the returned trajectory (Eq. 13b)
    for t in range(N):
        A, B, c = dyn(sc, 0, t)
        assert np.abs(o.s[0, t + 1] - (A @ o.s[0, t] + B @ o.u[0, t] + c)).max() <= 1e-12 * (1 + np.abs(o.s).max())


def test_multiplier_spec_example(orc):
    (inp, exp), = golden("multiplier")
    zeta0, T = inp
    sc = scenes.make_config(1)
    o = orc.Oracle(sc)
    # lambda = e_e / b_e, mu = 0, gamma = T - 1  =>  T_p = 1 + gamma = T,  R_p = a_e / b_e
    nr = 4
    e = int(np.argmax(sc.part_b))
    o.y[:] = 0
    o.y[:, e] = 1.0 / sc.part_b[e]
    o.y[:, nr + 4] = T - 1.0
    o.zeta[:] = zeta0
    o.multiplier_update()
    np.testing.assert_allclose(o.zeta, exp[0], rtol=1e-15)


def test_multiplier_zero_on_duality_certificates(orc):
    """For a separated pair, an optimal dual-LP solution (Eq. 5, scipy HiGHS) with
    gamma = alpha* - 1 makes T = R = 0 (Eqs. 10-11), so zeta, xi stay put."""
    sc = scenes.make_config(2)
    o = orc.Oracle(sc)
    o.admm_iterate(20)
    o.zeta[:] = 0.0
    o.xi[:] = 0.0
    N, M, d = sc.horizon, sc.n_obs, sc.dim
    sep = []
    p = 0
    for t in range(1, N + 1):
        R, rho = pose_of(sc, o.s[0, t])
        A, bb = sc.part_A, sc.part_b
        for j in range(M):
            Cm = sc.obs_C[sc.obs_off[j]:sc.obs_off[j + 1]]
            dv = sc.obs_d[sc.obs_off[j]:sc.obs_off[j + 1]]
            nr, no = len(bb), len(dv)
            Aeq = np.zeros((1 + d, nr + no))
            Aeq[0, :nr] = bb
            Aeq[1:, :nr] = A.T
            Aeq[1:, nr:] = (Cm @ R).T
            res = linprog(np.r_[np.zeros(nr), dv - Cm @ rho], A_eq=Aeq, b_eq=np.r_[1.0, np.zeros(d)],
                          bounds=[(0, None)] * (nr + no), method="highs")
            alpha = -res.fun
            if alpha > 1 + 1e-6:
                o.y[p, :nr + no] = res.x
                o.y[p, nr + no] = alpha - 1
                sep.append(p)
            p += 1
    assert len(sep) > 20
    o.multiplier_update()
    assert np.abs(o.zeta[sep]).max() < 1e-9
    assert np.abs(o.xi[sep]).max() < 1e-9


def translate_scene(sc, delta):
    d = sc.dim
    ds = np.zeros(sc.n_state)
    ds[sc.pose_idx[:d]] = delta
    dA = sc.dyn_A
    c = sc.dyn_c + ds[None] - np.einsum("tij,j->ti", dA, ds)
    return dataclasses.replace(sc, obs_d=sc.obs_d + sc.obs_C @ delta, s0=sc.s0 + ds, s_ref=sc.s_ref + ds,
                               dyn_c=c), ds


@pytest.mark.parametrize("cfg", [2, 11])
def test_translation_equivariance(orc, cfg):
    sc = scenes.make_config(cfg)
    a = orc.Oracle(sc)
    a.admm_iterate(sc.iters)
    sc2, ds = translate_scene(sc, np.array([3.7, -1.2]))
    b = orc.Oracle(sc2)
    b.admm_iterate(sc.iters)
    np.testing.assert_allclose(b.s - ds, a.s, atol=1e-7)
    np.testing.assert_allclose(b.u, a.u, atol=1e-7)


def test_obstacle_permutation_invariance(orc):
    sc = scenes.make_config(2)
    a = orc.Oracle(sc)
    a.admm_iterate(sc.iters)
    perm = [2, 0, 3, 1]
    sc2 = dataclasses.replace(sc)
    offs, Cs, ds_ = [0], [], []
    for j in perm:
        lo, hi = sc.obs_off[j], sc.obs_off[j + 1]
        Cs.append(sc.obs_C[lo:hi])
        ds_.append(sc.obs_d[lo:hi])
        offs.append(offs[-1] + hi - lo)
    sc2.obs_off, sc2.obs_C, sc2.obs_d = np.array(offs, np.int32), np.concatenate(Cs), np.concatenate(ds_)
    b = orc.Oracle(sc2)
    b.admm_iterate(sc.iters)
    np.testing.assert_allclose(b.s, a.s, atol=1e-8)
    np.testing.assert_allclose(b.u, a.u, atol=1e-8)
