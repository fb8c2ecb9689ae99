"""GPU (C-ABI, libca.so on a B200) vs the CPU oracle, on the same seeded inputs.

T1 frozen inputs: one ADMM step from an identical iterate -- per-pair y within
1e-9 (relative), identical pivot counts / status except rare near-tie Lemke
flips which are validated (unique u* and optimum, KKT certificate); primal and
multiplier steps within 1e-9.  T2: K full iterations on C1-C4 within 1e-6.
C5 at full size in the bench launch configuration: every iteration of sampled
scenes checked step by step against the oracle.  Plus scale detection, edge
cases (no obstacles, n > 16, d = 3), bitwise run-to-run and fused == stepwise.
"""
import dataclasses

import numpy as np
import pytest

import oracle
import scenes
from conftest import poly_from_vertices
from parity_util import compare_dual_sweep

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ca():
    from paper_2406_07048_b200 import build

    build.build()
    import paper_2406_07048_b200 as ca

    return ca


def scene(cfg):
    if cfg == 5:
        return scenes.make_c5(scene_ids=[0, 1777, 4095])
    return scenes.make_config(cfg)


def warm(sc, k0):
    o = oracle.Oracle(sc)
    if k0:
        o.admm_iterate(k0)
    return o


def close(a, b, rtol, what):
    a, b = np.asarray(a), np.asarray(b)
    err = np.abs(a - b) / np.maximum(1.0, np.abs(b))
    assert err.max() <= rtol, f"{what}: max rel err {err.max():.3e} at {np.unravel_index(err.argmax(), err.shape)}"


@pytest.mark.parametrize("cfg", [1, 2, 3, 4, 5, 6, 9, 10, 11, 12])
@pytest.mark.parametrize("k0", [0, 3])
def test_t1_dual_sweep(ca, cfg, k0):
    sc = scene(cfg)
    o = warm(sc, k0)
    g = ca.Problem(sc)
    g.set_iterate(o.s, o.u, o.y, o.zeta, o.xi)
    s, zeta, xi = o.s.copy(), o.zeta.copy(), o.xi.copy()
    rc, r = g.dual_sweep()
    rd, fails = o.dual_sweep()
    st = g.pair_state()
    flips = compare_dual_sweep(sc, s, zeta, xi, st["y"], o.y, st["pivots"], o.pivots, st["status"], o.status)
    assert r.n_fail == fails
    assert r.pivots == o.pivots.sum() or flips
    if not flips:
        close(r.r_dual, rd.sum(), 1e-9, "r_dual")
    # zeta, xi untouched by step 1
    assert np.array_equal(st["zeta"], zeta) and np.array_equal(st["xi"], xi)


@pytest.mark.parametrize("cfg", [1, 2, 3, 4, 6, 7, 8, 9, 10, 11, 12])
def test_t1_primal_and_multiplier(ca, cfg):
    sc = scene(cfg)
    o = warm(sc, 3)
    g = ca.Problem(sc)
    g.set_iterate(o.s, o.u, o.y, o.zeta, o.xi)
    o.set_iterate()  # both box blocks restart from w = Pi_box(s, u), l = 0 (C2b)
    g.dual_sweep()
    o.dual_sweep()
    s_lin = o.s.copy()  # dyn_model 1 linearises here
    g.primal_step()
    o.primal_step()
    s, u = g.trajectory()
    close(s, o.s, 1e-9, "s after primal step")
    close(u, o.u, 1e-9, "u after primal step")
    r = g.multiplier_update()
    rp = o.multiplier_update()
    st = g.pair_state()
    scale = 1.0 + np.abs(o.zeta).max()
    assert np.abs(st["zeta"] - o.zeta).max() <= 1e-9 * scale
    assert np.abs(st["xi"] - o.xi).max() <= 1e-9 * scale
    close(r.r_pri, rp.sum(), 1e-8, "r_pri")
    # dynamics hold exactly (Eq. 13b)
    sc0 = sc
    if sc0.dyn_model == 1:  # the unicycle linearised at the pre-step iterate
        dA, dB, dc = scenes.unicycle_ltv(s_lin[0, :sc0.horizon], sc0.dt)
    for t in range(sc0.horizon):
        k = t if sc0.dyn_per_time else 0
        if sc0.dyn_model == 1:
            A, B, c = dA[t], dB[t], dc[t]
        else:
            A, B, c = sc0.dyn_A[k], sc0.dyn_B[k], sc0.dyn_c[k]
        assert np.abs(s[0, t + 1] - (A @ s[0, t] + B @ u[0, t] + c)).max() <= 1e-12 * (1 + np.abs(s).max())


@pytest.mark.parametrize("cfg", [1, 2, 3, 4, 6, 7, 8, 9, 10, 11, 12])
def test_t2_full_iterations(ca, cfg):
    sc = scene(cfg)
    K = sc.iters
    g = ca.Problem(sc)
    rc, hist = g.admm_iterate(K)
    o = oracle.Oracle(sc)
    hp, hd, fails = o.admm_iterate(K)
    s, u = g.trajectory()
    close(s, o.s, 1e-6, "s")
    close(u, o.u, 1e-6, "u")
    # per entry of the residual histories, 1e-6 max(1, |r_orc|)
    close(hist["r_pri"], hp.sum(1), 1e-6, "r_pri history")
    close(hist["r_dual"], hd.sum(1), 1e-6, "r_dual history")
    assert hist["n_fail"].sum() == fails == 0
    st = g.pair_state()
    scale = 1.0 + np.abs(o.zeta).max()
    assert np.abs(st["zeta"] - o.zeta[: g.n_pairs]).max() <= 1e-6 * scale


def test_fused_pipeline_equals_stepwise_bitwise(ca):
    sc = scene(2)
    a = ca.Problem(sc)
    a.admm_iterate(12)
    b = ca.Problem(sc)
    for _ in range(12):
        b.admm_iterate(1)
    sa, ua = a.trajectory()
    sb, ub = b.trajectory()
    pa, pb = a.pair_state(), b.pair_state()
    assert np.array_equal(sa, sb) and np.array_equal(ua, ub)
    for k in ("y", "zeta", "xi", "pivots"):
        assert np.array_equal(pa[k], pb[k]), k


@pytest.mark.parametrize("cfg", [5, 1, 3, 4, 8, 12])
def test_run_to_run_bitwise(ca, cfg):
    """Fresh handles, same inputs: bitwise identical results (no atomics in any
    floating-point reduction; every shared-memory exchange of the scan / warp
    recursion / dense Lemke properly synchronised)."""
    sc = scenes.make_c5(n_scenes=8) if cfg == 5 else scene(cfg)
    outs = []
    for _ in range(2):
        g = ca.Problem(sc)
        rc, h = g.admm_iterate(10)
        outs.append((g.trajectory(), g.pair_state(), h))
    (s1, u1), p1, h1 = outs[0]
    (s2, u2), p2, h2 = outs[1]
    assert np.array_equal(s1, s2) and np.array_equal(u1, u2)
    assert np.array_equal(p1["y"], p2["y"]) and np.array_equal(h1["r_pri"], h2["r_pri"])


@pytest.mark.parametrize("cfg", [1, 2, 3, 4, 5, 6, 10, 11, 12])
def test_scale_detect(ca, cfg):
    sc = scene(cfg)
    o = warm(sc, 5)
    g = ca.Problem(sc)
    for states in (sc.s_ref, o.s):
        a_g, amin = g.scale_detect(states)
        a_o = o.scale_detect(states)
        close(a_g, a_o, 1e-9, "alpha*")
        per = a_o.reshape(sc.n_scenes, -1).min(1)
        close(amin, per, 1e-9, "min alpha")


def test_zero_obstacles(ca):
    sc = scenes.make_config(2)
    sc = dataclasses.replace(sc, n_obs=0, obs_off=np.zeros(1, np.int32), obs_C=np.zeros((0, 2)),
                             obs_d=np.zeros(0))
    g = ca.Problem(sc)
    g.admm_iterate(2)
    o = oracle.Oracle(sc)
    o.admm_iterate(2)
    s, u = g.trajectory()
    close(s, o.s, 1e-9, "s")
    close(u, o.u, 1e-9, "u")


def many_faced_scene(nv_lo=14, nv_hi=22, n_obs=6, seed=99):
    """C1-like car scene whose obstacles have 14-22 faces: n up to 27 (NMAX=32 path)."""
    rng = np.random.default_rng(seed)
    base = scenes.make_config(2)
    polys = []
    for k in range(n_obs):
        nv = int(rng.integers(nv_lo, nv_hi + 1))
        ang = 2 * np.pi * np.arange(nv) / nv + rng.uniform(-0.1, 0.1, nv) + rng.uniform(0, 6.28)
        r = rng.uniform(0.8, 2.0)
        c = np.array([4.0 + 2.2 * k, rng.uniform(-1.5, 1.5)])
        V = c + r * np.stack([np.cos(ang), np.sin(ang)], 1)
        polys.append(poly_from_vertices(V))
    off = np.concatenate([[0], np.cumsum([len(p[1]) for p in polys])]).astype(np.int32)
    return dataclasses.replace(base, n_obs=n_obs, obs_off=off, obs_C=np.concatenate([p[0] for p in polys]),
                               obs_d=np.concatenate([p[1] for p in polys]), iters=40)


def test_large_n_path(ca):
    sc = many_faced_scene()
    assert sc.n_max > 20
    o = warm(sc, 3)
    g = ca.Problem(sc)
    g.set_iterate(o.s, o.u, o.y, o.zeta, o.xi)
    s, zeta, xi = o.s.copy(), o.zeta.copy(), o.xi.copy()
    g.dual_sweep()
    o.dual_sweep()
    st = g.pair_state()
    compare_dual_sweep(sc, s, zeta, xi, st["y"], o.y, st["pivots"], o.pivots, st["status"], o.status)
    g2 = ca.Problem(sc)
    g2.admm_iterate(sc.iters)
    o2 = oracle.Oracle(sc)
    o2.admm_iterate(sc.iters)
    s2, u2 = g2.trajectory()
    close(s2, o2.s, 1e-6, "s (large n)")


def test_c5_full_size_stepwise(ca):
    """C5 at BASELINE size (4096 scenes x 200 obstacles x N=50) in the bench's launch
    configuration; sampled scenes are followed iteration by iteration: each GPU
    iteration equals the oracle's iteration applied to the GPU's previous iterate
    (non-unique Lemke choices validated, then adopted, reading #2)."""
    sc = scenes.make_c5()
    g = ca.Problem(sc)
    K = 12
    samples = [0, 2049, 4095]
    per = sc.horizon * sc.n_parts * sc.n_obs
    subs = {b: sc.subset([b]) for b in samples}

    def grab(b):
        s, u = g.trajectory()
        st = g.pair_state(b * per, per)
        return s[b:b + 1], u[b:b + 1], st

    prev = {b: grab(b) for b in samples}
    total_flips = 0
    for k in range(K):
        g.admm_iterate(1)
        for b in samples:
            s0, u0, st0 = prev[b]
            o = oracle.Oracle(subs[b])
            o.set_iterate(s=s0, u=u0, y=st0["y"], zeta=st0["zeta"], xi=st0["xi"])
            o.dual_sweep()
            s1, u1, st1 = grab(b)
            total_flips += compare_dual_sweep(subs[b], s0, st0["zeta"], st0["xi"], st1["y"], o.y, st1["pivots"],
                                              o.pivots, st1["status"], o.status)
            o.y[...] = st1["y"]  # adopt the GPU's (validated) minimisers
            o.primal_step()
            # trajectory tolerance of BASELINE.json north_star (1e-6); measured ~1e-9 here
            # (Riccati vs dense Cholesky of an LQ with condition ~1e6, sigma = 300)
            close(s1, o.s, 1e-6, f"s scene {b} iter {k}")
            close(u1, o.u, 1e-6, f"u scene {b} iter {k}")
            o.multiplier_update()
            sc_z = 1 + np.abs(o.zeta).max()
            assert np.abs(st1["zeta"] - o.zeta).max() <= 1e-9 * sc_z
            assert np.abs(st1["xi"] - o.xi).max() <= 1e-9 * sc_z
            prev[b] = (s1, u1, st1)
    print("C5 validated Lemke flips:", total_flips)


@pytest.mark.parametrize("cfg", [2, 4, 6, 8, 9, 10])
def test_obstacle_sharded_world1_nccl(ca, cfg):
    """The obstacle-sharded path (record reduction + ncclAllReduce + replicated Riccati)
    at world size 1 matches the unsharded solve (summation order differs)."""
    sc = scene(cfg)
    K = 20
    a = ca.Problem(sc)
    rca, ha = a.admm_iterate(K)
    b = ca.Problem(sc, dist=(1, 0, ca.nccl_unique_id()))
    rcb, hb = b.admm_iterate(K)
    sa, ua = a.trajectory()
    sb, ub = b.trajectory()
    close(sb, sa, 1e-10, "s (sharded vs plain)")
    close(ub, ua, 1e-10, "u (sharded vs plain)")
    np.testing.assert_allclose(hb["r_pri"], ha["r_pri"], rtol=1e-9, atol=1e-12)
    np.testing.assert_allclose(hb["r_dual"], ha["r_dual"], rtol=1e-9, atol=1e-12)
    _, ma = a.scale_detect(want_alpha=False)
    _, mb = b.scale_detect(want_alpha=False)
    np.testing.assert_allclose(mb, ma, rtol=1e-12)


def symmetric_scene():
    """Degenerate geometry: an obstacle with a duplicated face (two identical LCP rows:
    exact ratio-test ties -> the lexicographic rule, solved by the warp-cooperative
    dense re-solve), obstacles centred on the reference line, one touching the car
    at t = 0, a diamond whose vertex points at the car."""
    def dup(poly):  # every face twice: exact ties between the copies' LCP rows
        return np.repeat(poly[0], 2, axis=0), np.repeat(poly[1], 2)

    polys = [
        dup(scenes.box_hrep([6.0, 0.0], [1.0, 1.0])),
        dup(scenes.box_hrep([10.0, 0.0], [0.5, 2.0])),
        scenes.polygon_hrep([14.0, 0.0], 1.5, np.array([0.0, 0.5, 1.0, 1.5]) * np.pi),
        scenes.box_hrep([3.25, 0.0], [1.0, 1.0]),  # face at x = 2.25: touches the car body at t = 0
    ]
    return scenes._car_common("SYM", 0, 0, N=20, iters=20, speed=4.0, polys_per_scene=[polys])


@pytest.mark.parametrize("mode", ["auto", "revised"])
@pytest.mark.parametrize("k0", [0, 2, 6])
def test_t1_symmetric_degenerate(ca, k0, mode, monkeypatch):
    """auto: this small problem runs the latency mode (every pair dense); revised: the
    one-thread revised path, whose lexicographic ties go to the dense re-solve."""
    if mode == "revised":
        monkeypatch.setenv("CA_SWEEP_DENSE", "0")
    sc = symmetric_scene()
    o = warm(sc, k0)
    g = ca.Problem(sc)
    g.set_iterate(o.s, o.u, o.y, o.zeta, o.xi)
    s, zeta, xi = o.s.copy(), o.zeta.copy(), o.xi.copy()
    rc, r = g.dual_sweep()
    o.dual_sweep()
    st = g.pair_state()
    compare_dual_sweep(sc, s, zeta, xi, st["y"], o.y, st["pivots"], o.pivots, st["status"], o.status)
    # the duplicated faces produce lexicographic ties, re-solved by the dense path
    assert np.count_nonzero(st["status"] & 0x100) > 0


@pytest.mark.parametrize("mode", ["auto", "revised"])
def test_t2_symmetric_degenerate(ca, mode, monkeypatch):
    if mode == "revised":
        monkeypatch.setenv("CA_SWEEP_DENSE", "0")
    sc = symmetric_scene()
    g = ca.Problem(sc)
    o = oracle.Oracle(sc)
    K = 20
    rc, h = g.admm_iterate(K)
    o.admm_iterate(K)
    s, u = g.trajectory()
    close(s, o.s, 1e-6, "s")
    close(u, o.u, 1e-6, "u")


@pytest.mark.parametrize("cfg", [2, 5])
def test_torch_workspace_bitwise(ca, cfg):
    """Every device buffer carved out of one torch tensor (ca_workspace_size bytes):
    the same results bit for bit as library-allocated memory."""
    sc = scene(cfg)
    a = ca.Problem(sc)
    b = ca.Problem(sc, workspace="torch")
    assert b._ws.numel() >= b.device_bytes > 0
    a.admm_iterate(10)
    b.admm_iterate(10)
    (sa, ua), (sb, ub) = a.trajectory(), b.trajectory()
    assert np.array_equal(sa, sb) and np.array_equal(ua, ub)
    pa, pb = a.pair_state(), b.pair_state()
    for k in ("y", "zeta", "xi", "pivots", "status"):
        assert np.array_equal(pa[k], pb[k]), k
    aa, ma = a.scale_detect()
    ab, mb = b.scale_detect()
    assert np.array_equal(aa, ab) and np.array_equal(ma, mb)


def test_box_block_parity(ca):
    """NEXT f1 (reading #7): the box block's w, l and residual after K iterations,
    then one more primal step from the same (nonzero-l) state, against the oracle."""
    sc = scenes.make_config(8)
    g = ca.Problem(sc)
    o = oracle.Oracle(sc)
    ws, ls, wu, lu, res = g.box_state()  # cold start: iterate projected into the box
    s, u = g.trajectory()
    np.testing.assert_array_equal(s, o.s)
    np.testing.assert_array_equal(u, o.u)
    np.testing.assert_array_equal(ws, o.ws)
    assert not ls.any() and not lu.any() and not res.any()
    g.admm_iterate(6)
    o.admm_iterate(6)
    ws, ls, wu, lu, res = g.box_state()
    for a, b, what in ((ws, o.ws, "w_s"), (ls, o.ls, "l_s"), (wu, o.wu, "w_u"), (lu, o.lu, "l_u")):
        close(a[:, 1:] if a.shape == o.ws.shape else a, b[:, 1:] if b.shape == o.ws.shape else b, 1e-8, what)
    assert np.abs(ls).max() > 1e-3 and np.abs(lu).max() > 1e-3  # the bounds are active
    close(res, o.boxres, 1e-8, "box residual")
    # the same state on both sides, then one primal step with l != 0
    s, u = g.trajectory()
    st = g.pair_state()
    o.s[...], o.u[...] = s, u
    o.y[: g.n_pairs], o.zeta[: g.n_pairs], o.xi[: g.n_pairs] = st["y"], st["zeta"], st["xi"]
    o.ws[...], o.ls[...], o.wu[...], o.lu[...] = ws, ls, wu, lu
    g.dual_sweep()
    o.dual_sweep()
    g.primal_step()
    o.primal_step()
    s, u = g.trajectory()
    close(s, o.s, 1e-9, "s after primal step (box)")
    close(u, o.u, 1e-9, "u after primal step (box)")
    ws, ls, wu, lu, res = g.box_state()
    close(ls[:, 1:], o.ls[:, 1:], 1e-9, "l_s after primal step")
    close(lu, o.lu, 1e-9, "l_u after primal step")
    close(res, o.boxres, 1e-8, "box residual after primal step")


def test_box_infinite_bounds_equal_unbounded_bitwise(ca):
    sc = scenes.make_config(2)
    inf = np.inf
    sb = dataclasses.replace(sc, s_min=np.full(4, -inf), s_max=np.full(4, inf), u_min=np.full(2, -inf),
                             u_max=np.full(2, inf), box_rho=5.0)
    a, b = ca.Problem(sc), ca.Problem(sb)
    ha = a.admm_iterate(20)[1]
    hb = b.admm_iterate(20)[1]
    sa, ua = a.trajectory()
    s2, u2 = b.trajectory()
    assert np.array_equal(sa, s2) and np.array_equal(ua, u2)
    assert np.array_equal(ha["r_pri"], hb["r_pri"])


def sensing_scenes():
    return {"c4s": scenes.make_config(9),
            "c5s": dataclasses.replace(scenes.make_c5(scene_ids=[0, 7, 4000]), sense_half=np.array([25.0, 25.0])),
            "c3s": dataclasses.replace(scenes.make_config(3), sense_half=np.array([4.0, 1.0, 0.6]))}


@pytest.mark.parametrize("case", ["c4s", "c5s", "c3s"])
def test_sensing_mask_and_sweep(ca, case):
    """NEXT f3 sensing: the GPU's sensed set (k_sense, vertex enumeration) equals the
    oracle's (scale LP of the sensing box); unsensed pairs report alpha = +inf and are
    skipped by the dual step; one warm dual sweep matches pair by pair."""
    sc = sensing_scenes()[case]
    o = warm(sc, 2)
    g = ca.Problem(sc)
    alpha, _ = g.scale_detect(states=o.s)
    a_o = o.scale_detect()
    assert 0 < np.isfinite(a_o).sum() < a_o.size
    assert np.array_equal(np.isinf(alpha[: g.n_pairs]), np.isinf(a_o))
    fin = np.isfinite(a_o)
    close(alpha[: g.n_pairs][fin], a_o[fin], 1e-9, "alpha (sensed pairs)")
    g.set_iterate(o.s, o.u, o.y, o.zeta, o.xi)
    s, zeta, xi = o.s.copy(), o.zeta.copy(), o.xi.copy()
    rc, r = g.dual_sweep()
    rd, fails = o.dual_sweep()
    st = g.pair_state()
    flips = compare_dual_sweep(sc, s, zeta, xi, st["y"], o.y, st["pivots"], o.pivots, st["status"], o.status)
    assert r.n_fail == fails
    assert r.pivots == o.pivots.sum() or flips


def test_load_keeps_feature_presence(ca):
    """ca_problem_load refuses a problem whose optional features (boxes, sensing,
    scaling centres) differ from the handle's (their buffers are sized at create),
    and reloading the same kind of problem re-evaluates them (sensing from the new s0)."""
    sc = scenes.make_config(9)
    g = ca.Problem(sc)
    for bad in (dataclasses.replace(sc, sense_half=None),
                dataclasses.replace(sc, u_min=np.array([-1.0, -1.0]), u_max=np.array([1.0, 1.0]), box_rho=1.0)):
        with pytest.raises(ca.CAError):
            g.load(bad)
    moved = dataclasses.replace(sc, s0=sc.s0 + np.array([[150.0, 0.0, 0.0, 0.0]]))
    g.load(moved)
    alpha, _ = g.scale_detect()
    o = oracle.Oracle(moved)
    a_o = o.scale_detect()
    assert np.array_equal(np.isinf(alpha[: g.n_pairs]), np.isinf(a_o))
    assert not np.array_equal(np.isinf(a_o), np.isinf(oracle.Oracle(sc).scale_detect()))


@pytest.mark.parametrize("cfg", [1, 2, 3, 10])
def test_small_configs_revised_path(ca, cfg, monkeypatch):
    """Small problems run the latency mode (one pair per warp, dense Lemke) by default;
    the one-thread revised path on the same problems (CA_SWEEP_DENSE=0) against the
    oracle, and the latency mode's pivot counts equal to the oracle's exactly."""
    sc = scene(cfg)
    K = 30
    o = oracle.Oracle(sc)
    hp, hd, fails = o.admm_iterate(K)
    g = ca.Problem(sc)
    g.admm_iterate(K)
    assert np.array_equal(g.pair_state()["pivots"], o.pivots[: g.n_pairs])  # dense: the oracle's rules verbatim
    monkeypatch.setenv("CA_SWEEP_DENSE", "0")
    g = ca.Problem(sc)
    rc, hist = g.admm_iterate(K)
    s, u = g.trajectory()
    close(s, o.s, 1e-6, "s")
    close(u, o.u, 1e-6, "u")
    close(hist["r_pri"], hp.sum(1), 1e-6, "r_pri history")
    close(hist["r_dual"], hd.sum(1), 1e-6, "r_dual history")
    assert hist["n_fail"].sum() == fails == 0


@pytest.mark.parametrize("cfg", [8, 10])
def test_large_batch_paths_with_features(ca, cfg):
    """Large batches (> 1024 scenes) take the thread-per-scene Riccati and the pooled
    revised sweep: with boxes (C2b) and scaling centres (C2t) every scene of a
    replicated batch must match the single-scene oracle."""
    sc1 = scenes.make_config(cfg)
    big = sc1.subset([0] * 1025)
    K = 10
    g = ca.Problem(big)
    g.admm_iterate(K)
    s, u = g.trajectory()
    o = oracle.Oracle(sc1)
    o.admm_iterate(K)
    for b in (0, 511, 1024):
        close(s[b], o.s[0], 1e-8, f"s scene {b}")
        close(u[b], o.u[0], 1e-8, f"u scene {b}")
    if cfg == 8:
        ws, ls, wu, lu, res = g.box_state()
        close(lu[1024], o.lu[0], 1e-8, "l_u")
        close(res[1024:], o.boxres, 1e-8, "box residual")


def test_sensing_pooled_sweep(ca):
    """Sensing through the pooled sweep (800-pair sort pools over 4 timesteps, 256
    scenes): sampled scenes against the single-scene oracle after K iterations."""
    big = dataclasses.replace(scenes.make_c5(n_scenes=256), sense_half=np.array([20.0, 20.0]))
    K = 3
    g = ca.Problem(big)
    g.admm_iterate(K)
    s, u = g.trajectory()
    for b in (0, 97, 255):
        one = big.subset([b])
        o = oracle.Oracle(one)
        assert 0 < o.sensed.sum() < o.sensed.size
        o.admm_iterate(K)
        close(s[b], o.s[0], 1e-8, f"s scene {b}")
        close(u[b], o.u[0], 1e-8, f"u scene {b}")


@pytest.mark.parametrize("cfg", [1, 2, 3, 4])
def test_prox_regularised_parity(ca, cfg):
    """prox_eps > 0 (reading #2): (eps/2)||y - y^k||^2 makes every pair QP strictly
    convex; the GPU solves it with the dense Lemke on M + eps (I + kt kt^T).  One warm
    dual sweep pair by pair (y and pivot counts) and K full iterations vs the oracle."""
    eps = 1e-2
    sc = scene(cfg)
    o = oracle.Oracle(sc, prox_eps=eps)
    o.admm_iterate(3)
    g = ca.Problem(sc, prox_eps=eps, prox_solver=1)
    g.set_iterate(o.s, o.u, o.y, o.zeta, o.xi)
    rc, r = g.dual_sweep()
    o.dual_sweep()
    st = g.pair_state()
    close(st["y"], o.y[: g.n_pairs], 1e-9, "y (prox)")
    assert np.array_equal(st["pivots"], o.pivots[: g.n_pairs])
    K = 20
    g = ca.Problem(sc, prox_eps=eps, prox_solver=1)
    g.admm_iterate(K)
    o = oracle.Oracle(sc, prox_eps=eps)
    hp, hd, fails = o.admm_iterate(K)
    s, u = g.trajectory()
    close(s, o.s, 1e-6, "s (prox)")
    close(u, o.u, 1e-6, "u (prox)")


def prox_rtol(sc, eps):
    """Tolerance for two different exact solvers of the prox pair QP: 4 ulp x the
    condition number 1 + ||K||^2 / eps of its Hessian in y, with the unit-row bound
    ||K_k|| <= 1 + |d_l| + |rho - t step| (Eq. 19b rows), floored at T1's 1e-9."""
    d = sc.dim
    pos = np.abs(sc.s_ref[..., [int(i) for i in sc.pose_idx[:d]]]).max()
    step = getattr(sc, "obs_step", None)
    if step is not None:
        pos += sc.horizon * np.abs(step).max()
    kmax = 1.0 + np.abs(sc.obs_d).max() + pos
    return max(1e-9, 4e-16 * (1.0 + kmax * kmax / eps))


@pytest.mark.parametrize("cfg", [1, 2, 3, 4, 6, 7, 8, 9, 10])
@pytest.mark.parametrize("eps", [1e-3, 1e-1])
def test_prox_newton_parity(ca, cfg, eps):
    """NEXT f4: the dual semismooth Newton solver (prox_solver 0, one pair per thread)
    returns the unique minimiser of the prox-regularised pair QP (reading #2), which the
    oracle computes with the dense Lemke.  Different algorithms, so agreement is to the
    rounding of the QP's conditioning: y to prox_rtol (the Hessian in y has condition
    <= 1 + ||K||^2 / eps), whole ADMM runs (s, u after K iterations) to 1e-6 as T2."""
    sc = scene(cfg)
    o = oracle.Oracle(sc, prox_eps=eps)
    o.admm_iterate(3)
    g = ca.Problem(sc, prox_eps=eps)
    g.set_iterate(o.s, o.u, o.y, o.zeta, o.xi)
    g.dual_sweep()
    o.dual_sweep()
    st = g.pair_state()
    close(st["y"], o.y[: g.n_pairs], prox_rtol(sc, eps), "y (prox, Newton)")
    assert np.all(st["status"] & 15 == 0)  # solved (a Newton non-convergence -> dense re-solve, bit 4)
    K = 20
    g = ca.Problem(sc, prox_eps=eps)
    g.admm_iterate(K)
    o = oracle.Oracle(sc, prox_eps=eps)
    o.admm_iterate(K)
    s, u = g.trajectory()
    close(s, o.s, 1e-6, "s (prox, Newton)")
    close(u, o.u, 1e-6, "u (prox, Newton)")


def test_prox_newton_c5_sample(ca):
    """NEXT f4 at batch scale: 64 C5 scenes through the Newton solver; sampled scenes
    against the single-scene oracle after K iterations, and against the dense-Lemke
    GPU path on the whole batch."""
    eps = 1e-2
    big = scenes.make_c5(n_scenes=64)
    K = 3
    g = ca.Problem(big, prox_eps=eps)
    g.admm_iterate(K)
    s, u = g.trajectory()
    h = ca.Problem(big, prox_eps=eps, prox_solver=1)
    h.admm_iterate(K)
    s1, u1 = h.trajectory()
    close(s, s1, 1e-7, "s Newton vs dense Lemke")
    close(u, u1, 1e-7, "u Newton vs dense Lemke")
    for b in (0, 41):
        o = oracle.Oracle(big.subset([b]), prox_eps=eps)
        o.admm_iterate(K)
        close(s[b], o.s[0], 1e-7, f"s scene {b}")
        close(u[b], o.u[0], 1e-7, f"u scene {b}")
