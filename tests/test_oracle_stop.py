"""Pins of Eq. 18 in the oracle: the primal and dual residual sums
recomputed in numpy from consecutive iterates, the '<=' stopping test (SPEC S:526-528
worked examples, monotone in eps), the per-scene ADMM-until-Eq.-18 loop, and
the threaded fan-out used for the all-core CPU baseline.

r_pri  = sum_ijt ||zeta^{k+1} - zeta^k||^2 + ||xi^{k+1} - xi^k||^2          (18a)
r_dual = sum_ijt ||lambda^{k+1} - lambda^k||^2 + ||mu^{k+1} - mu^k||^2        (18b)
per scene, raw sums (readings #19, #20: gamma excluded, no averaging); the box block's
||x - w||^2 joins r_pri (reading #7).  The oracle forms r_pri from T_p (Eq. 17's
increment) and r_dual from y^{k+1} - y^k inside its loops; the numpy side below takes
differences of the stored iterates, so a dropped gamma exclusion, an average, norms
instead of squares or a wrong block would all fail."""
import numpy as np
import pytest

import scenes
from test_oracle_scale import golden

U = 2.0 ** -53  # unit roundoff


def lcp_rows(sc):
    """per pair: n_r(i) + n_o(b, j) = the lambda and mu entries of y (gamma excluded)"""
    return sc.lcp_sizes() - 1


def scene_of_pair(sc):
    return np.repeat(np.arange(sc.n_scenes), sc.n_pairs // max(1, sc.n_scenes))


def case(name):
    if name == "c5x3":
        return scenes.make_c5(scene_ids=[0, 7, 11])
    return scenes.make_config(int(name[1:]))


CASES = ["c2", "c4", "c5x3", "c8", "c10", "c11", "c12"]


@pytest.mark.parametrize("name", CASES)
def test_residual_sums_recomputed(orc, name):
    sc = case(name)
    o = orc.Oracle(sc)
    o.admm_iterate(3)
    rows = lcp_rows(sc)
    sid = scene_of_pair(sc)
    mask = np.arange(o.ny)[None, :] < rows[:, None]  # lambda, mu entries of each pair
    # (18b) from y before / after the dual step
    y0 = o.y.copy()
    rd, fails = o.dual_sweep()
    dy = np.where(mask, o.y[: sc.n_pairs] - y0[: sc.n_pairs], 0.0)
    rd_np = np.bincount(sid, weights=(dy * dy).sum(1), minlength=sc.n_scenes)
    assert np.allclose(rd, rd_np, rtol=1e-12, atol=0.0), (rd, rd_np)
    # the gamma entry moved too, and is NOT in the sum (reading #19)
    g = np.take_along_axis(o.y[: sc.n_pairs] - y0[: sc.n_pairs], rows[:, None], 1)[:, 0]
    if np.any(g != 0.0):
        with_g = rd_np + np.bincount(sid, weights=g * g, minlength=sc.n_scenes)
        assert not np.allclose(rd, with_g, rtol=1e-12, atol=0.0)
    o.primal_step()
    # (18a) from zeta, xi before / after the multiplier step
    z0, x0 = o.zeta.copy(), o.xi.copy()
    rp = o.multiplier_update()
    dz = o.zeta[: sc.n_pairs] - z0[: sc.n_pairs]
    dx = o.xi[: sc.n_pairs] - x0[: sc.n_pairs]
    terms = dz * dz + (dx * dx).sum(1)
    rp_np = np.bincount(sid, weights=terms, minlength=sc.n_scenes)
    # zeta^{k+1} = fl(zeta^k + T): the stored difference differs from T by <= u |zeta^{k+1}|
    err = (2 * np.abs(dz) + U * np.abs(o.zeta[: sc.n_pairs])) * U * np.abs(o.zeta[: sc.n_pairs])
    err += ((2 * np.abs(dx) + U * np.abs(o.xi[: sc.n_pairs])) * U * np.abs(o.xi[: sc.n_pairs])).sum(1)
    tol = np.bincount(sid, weights=err, minlength=sc.n_scenes) + 1e-13 * rp_np
    if sc.s_min is not None or sc.u_min is not None:  # reading #7: + sum ||x - w||^2 of the box block
        inf = np.inf
        smin = np.full(sc.n_state, -inf) if sc.s_min is None else sc.s_min
        smax = np.full(sc.n_state, inf) if sc.s_max is None else sc.s_max
        umin = np.full(sc.n_ctrl, -inf) if sc.u_min is None else sc.u_min
        umax = np.full(sc.n_ctrl, inf) if sc.u_max is None else sc.u_max
        bs = np.isfinite(smin) | np.isfinite(smax)
        bu = np.isfinite(umin) | np.isfinite(umax)
        es = (o.s[:, 1:, :] - o.ws[:, 1:, :])[..., bs]
        eu = (o.u - o.wu)[..., bu]
        rp_np = rp_np + (es ** 2).sum((1, 2)) + (eu ** 2).sum((1, 2))
    assert np.all(np.abs(rp - rp_np) <= tol + 1e-13 * np.abs(rp_np)), (rp, rp_np, tol)


def test_stopping_spec_examples(orc):
    for inp, exp in golden("stopping"):
        assert orc.check_stopping(*inp) == bool(exp[0]), (inp, exp)


def test_stopping_monotone_in_eps(orc):
    """if Eq. 18 holds at (eps_pri, eps_dual) it holds at larger thresholds;
    and it is exactly the conjunction of the two '<=' tests."""
    rng = np.random.default_rng(18)
    for _ in range(2000):
        rp, rd, ep, ed = np.exp(rng.uniform(-5, 5, 4))
        if rng.uniform() < 0.2:
            ep = rp  # the '<=' boundary
        s = orc.check_stopping(rp, rd, ep, ed)
        assert s == ((rp <= ep) and (rd <= ed))
        if s:
            assert orc.check_stopping(rp, rd, ep * (1 + rng.uniform()), ed * (1 + rng.uniform()))


@pytest.mark.parametrize("name,eps,kmax", [("c1", None, 50), ("c2", None, 200), ("c8", None, 200),
                                           ("c11", None, 200), ("c5x2", 3.0, 40)])
def test_admm_solve_is_first_hit(orc, name, eps, kmax):
    """Per scene, admm_solve stops at the first iteration of the fixed-K history that
    meets Eq. 18 and leaves that scene's iterate there: equal (bitwise) to a fresh run
    of exactly that many fixed iterations."""
    sc = scenes.make_c5(scene_ids=[2, 3]) if name == "c5x2" else case(name)
    pps = sc.n_pairs // sc.n_scenes
    e = 1e-3 * pps if eps is None else eps  # SURVEY c.3 #12 default
    ref = orc.Oracle(sc)
    hp, hd, _ = ref.admm_iterate(kmax)
    o = orc.Oracle(sc)
    it, cv, rp, rd, _ = o.admm_solve(e, e, kmax)
    for b in range(sc.n_scenes):
        hit = [k for k in range(kmax) if hp[k, b] <= e and hd[k, b] <= e]
        want = hit[0] + 1 if hit else kmax
        assert it[b] == want and cv[b] == bool(hit), (b, it[b], want)
        assert rp[b] == hp[want - 1, b] and rd[b] == hd[want - 1, b]
        one = orc.Oracle(sc.subset([b]))
        one.admm_iterate(int(want))
        assert np.array_equal(one.s[0], o.s[b]) and np.array_equal(one.u[0], o.u[b])
    if name in ("c1", "c2", "c11"):
        assert cv.all()  # these converge under the default thresholds
    if name == "c5x2":
        assert list(cv) == [True, False]  # one scene stops early, the other runs to kmax


def test_threaded_fanout(orc):
    sc = scenes.make_c5(scene_ids=[3, 4, 5, 6, 7])
    a, b = orc.Oracle(sc), orc.Oracle(sc)
    hp, hd, _ = a.admm_iterate(3)
    hp2, hd2, _ = b.admm_iterate_mt(3, 2)  # scene fan-out: bitwise the sequential run
    assert np.array_equal(hp, hp2) and np.array_equal(hd, hd2) and np.array_equal(a.s, b.s)
    sc = scenes.make_config(2)
    a, b = orc.Oracle(sc), orc.Oracle(sc)
    hp, hd, _ = a.admm_iterate(5)
    hp2, hd2, _ = b.admm_iterate_mt(5, 3)  # pair fan-out: r_dual summed per range
    assert np.array_equal(a.y, b.y) and np.array_equal(a.s, b.s) and np.array_equal(hp, hp2)
    assert np.allclose(hd, hd2, rtol=1e-13, atol=0.0)
