"""GPU (libca.so through the C ABI) vs the CPU oracle for the rest of the hot path's
contract: ca_admm_solve (Eq. 18 per scene) against orc_admm_solve, the '<='
boundary, the per-kind failure counters of ca_residuals, the obstacle-sharded exchange
(a5) emulated on one GPU, scene sharding's independence, empty slices, and C5 T2 end to
end on 16 sampled scenes with the Lemke basis-agreement rate.
"""
import dataclasses
import os
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import pytest

import oracle
import scenes
from parity_util import pair_geometry

pytestmark = pytest.mark.gpu
NCPU = max(1, min(32, os.cpu_count() or 1))


@pytest.fixture(scope="module")
def ca():
    from paper_2406_07048_b200 import build

    build.build()
    import paper_2406_07048_b200 as ca

    return ca


def close(a, b, rtol, what):
    a, b = np.asarray(a), np.asarray(b)
    err = np.abs(a - b) / np.maximum(1.0, np.abs(b))
    assert err.max() <= rtol, f"{what}: max rel err {err.max():.3e} at {np.unravel_index(err.argmax(), err.shape)}"


def pmap(fn, items):
    """oracle runs in parallel threads (ctypes releases the GIL inside the C oracle)"""
    with ThreadPoolExecutor(NCPU) as ex:
        return list(ex.map(fn, items))


def case(name):
    if name == "c5x16":
        return scenes.make_c5(scene_ids=[int(b) for b in np.linspace(0, 4095, 16)])
    return scenes.make_config(int(name[1:]))


def oracle_solve_per_scene(sc, eps, kmax):
    """orc_admm_solve scene by scene (scenes are independent: = the batched call)"""
    def one(b):
        o = oracle.Oracle(sc.subset([b]))
        it, cv, rp, rd, _ = o.admm_solve(eps, eps, kmax)
        return int(it[0]), bool(cv[0]), o.s[0].copy(), o.u[0].copy(), rp[0], rd[0]
    return pmap(one, range(sc.n_scenes))


# ---------------------------------------------------------------------------
# Eq. 18: ca_admm_solve vs orc_admm_solve
# ---------------------------------------------------------------------------

@pytest.mark.parametrize("name,eps,kmax", [("c1", None, 50), ("c2", None, 200), ("c8", None, 200),
                                           ("c11", None, 200), ("c5x16", 3.0, 100)])
def test_admm_solve_parity(ca, name, eps, kmax):
    """Per scene: the same stop iteration and converged flag as the oracle (Eq. 18 with
    '<='), the stopped iterate within T2's 1e-6.  A scene whose oracle residual passes
    an Eq. 18 threshold within 1e-6 relative at some iteration is a genuine near-tie of
    the stop test (the two sides differ at the 1e-9 level) and is only reported."""
    sc = case(name)
    pps = sc.n_pairs // sc.n_scenes
    e = 1e-3 * pps if eps is None else eps  # SURVEY c.3 #12 default
    g = ca.Problem(sc, eps_pri=e, eps_dual=e, max_iters=kmax)
    rc, rep, it_g, cv_g = g.admm_solve()
    s_g, u_g = g.trajectory()
    rp_g, rd_g = g.scene_residuals()
    orc = oracle_solve_per_scene(sc, e, kmax)
    # the oracle's residual histories decide which stop tests are near-ties
    def hist(b):
        o = oracle.Oracle(sc.subset([b]))
        hp, hd, _ = o.admm_iterate(orc[b][0])
        return hp[:, 0], hd[:, 0]
    hists = pmap(hist, range(sc.n_scenes))
    ties = 0
    for b in range(sc.n_scenes):
        it_o, cv_o, s_o, u_o, rp_o, rd_o = orc[b]
        hp, hd = hists[b]
        near = np.any(np.abs(hp - e) <= 1e-6 * e) or np.any(np.abs(hd - e) <= 1e-6 * e)
        if near:
            ties += 1
            continue
        assert it_g[b] == it_o and cv_g[b] == cv_o, (b, it_g[b], it_o, cv_g[b], cv_o)
        close(s_g[b], s_o, 1e-6, f"s scene {b}")
        close(u_g[b], u_o, 1e-6, f"u scene {b}")
        close(rp_g[b], rp_o, 1e-6, f"r_pri scene {b}")
        close(rd_g[b], rd_o, 1e-6, f"r_dual scene {b}")
    assert ties <= max(0, sc.n_scenes // 8)
    assert rep["iterations"] == int(it_g.max()) and rep["converged"] == bool(cv_g.all())
    assert (rc == 0) == bool(cv_g.all())
    print(f"{name}: iterations {list(it_g)}, converged {int(cv_g.sum())}/{sc.n_scenes}, stop-test near-ties {ties}")


def test_admm_solve_boundary_is_le(ca):
    """a residual sum exactly equal to eps stops the solve ('<=').  eps_pri
    is set to the GPU's own r_pri of a record-low iteration k0 (same arithmetic path as
    the solve: one iteration per call); the solve must stop exactly there."""
    sc = scenes.make_config(2)
    g = ca.Problem(sc)
    rp = []
    for _ in range(40):
        g.admm_iterate(1)
        rp.append(g.scene_residuals()[0][0])
    rp = np.array(rp)
    k0 = max(k for k in range(5, 40) if rp[k] < rp[:k].min())
    h = ca.Problem(sc, eps_pri=float(rp[k0]), eps_dual=1e300, max_iters=60)
    rc, rep, it, cv = h.admm_solve()
    assert it[0] == k0 + 1 and cv[0] and rep["r_pri"] == rp[k0]
    h2 = ca.Problem(sc, eps_pri=float(np.nextafter(rp[k0], 0.0)), eps_dual=1e300, max_iters=60)
    rc, rep2, it2, cv2 = h2.admm_solve()
    assert it2[0] > k0 + 1  # one ulp below: not met at k0 ('<', not '<=', would fail the first)


def test_admm_solve_scenes_independent(ca):
    """Per-scene stopping makes every scene's result independent of the others: the
    8-scene batch solve equals, bitwise, the union of two 4-scene solves (the 1-GPU
    emulation of a 2-way scene shard) -- iterations, flags, trajectories."""
    sc = scenes.make_c5(scene_ids=range(8))
    kw = dict(eps_pri=3.0, eps_dual=3.0, max_iters=40)
    g = ca.Problem(sc, **kw)
    _, _, it, cv = g.admm_solve()
    s, u = g.trajectory()
    assert 0 < cv.sum() < 8  # some stop, some run to max_iters
    for half in (range(0, 4), range(4, 8)):
        h = ca.Problem(sc.subset(half), **kw)
        _, _, it_h, cv_h = h.admm_solve()
        sh, uh = h.trajectory()
        assert np.array_equal(it_h, it[half.start:half.stop]) and np.array_equal(cv_h, cv[half.start:half.stop])
        assert np.array_equal(sh, s[half.start:half.stop]) and np.array_equal(uh, u[half.start:half.stop])
    # after a solve, ca_admm_iterate runs every scene again
    g.admm_iterate(1)


def test_solve_scenes_before_solve_is_invalid(ca):
    g = ca.Problem(scenes.make_config(1))
    import ctypes as C
    from paper_2406_07048_b200 import _ca
    it = np.empty(1, np.int32)
    rc = _ca.lib().ca_get_solve_scenes(g.h, it.ctypes.data, None)
    assert rc == -1


# ---------------------------------------------------------------------------
# ca_residuals: every field
# ---------------------------------------------------------------------------

def test_residual_fields_and_failure_kinds(ca):
    """n_fail = n_ray + n_iterlimit + n_neg_ye, each equal to the oracle's count of that
    status on identical inputs (a pivot cap of 1 x n forces ITER_LIMIT failures, SPEC
    S:290); pivots and max_pivots against the per-pair counts; ms_* with timing on."""
    sc = scenes.make_config(2)
    o = oracle.Oracle(sc, max_pivot_factor=1)
    o.admm_iterate(4)
    g = ca.Problem(sc, max_pivot_factor=1)
    g.set_iterate(o.s, o.u, o.y, o.zeta, o.xi)
    g.set_timing(True)
    rc, r = g.dual_sweep()
    o.dual_sweep()
    st = g.pair_state()
    assert np.array_equal(st["status"] & 0xff, o.status[: g.n_pairs])
    cnt = {k: int(np.count_nonzero(o.status == k)) for k in (oracle.RAY, oracle.ITER_LIMIT, oracle.NEG_YE)}
    assert cnt[oracle.ITER_LIMIT] > 0
    assert r.n_iterlimit == cnt[oracle.ITER_LIMIT] and r.n_ray == cnt[oracle.RAY] and r.n_neg_ye == cnt[oracle.NEG_YE]
    assert r.n_fail == r.n_ray + r.n_iterlimit + r.n_neg_ye
    assert r.pivots == int(st["pivots"].sum()) and r.max_pivots == int(st["pivots"].max())
    assert r.n_pairs == g.n_pairs and r.ms_sweep > 0.0
    assert rc == ca.CA_W_PAIR_FAILURES
    # the history of ca_admm_iterate, timing on: per-iteration milliseconds
    g = ca.Problem(sc)
    g.set_timing(True)
    rc, h = g.admm_iterate(5)
    assert np.all(h["ms_sweep"] > 0) and np.all(h["ms_riccati"] > 0) and np.all(h["max_pivots"] > 0)
    assert np.all(h["ms_mult"][:-1] == 0) and h["ms_mult"][-1] > 0  # standalone update after the last sweep only
    assert np.all(h["n_fail"] == h["n_ray"] + h["n_iterlimit"] + h["n_neg_ye"])


# ---------------------------------------------------------------------------
# multi-GPU paths on one GPU
# ---------------------------------------------------------------------------

def obstacle_half(sc, j0, j1):
    M = sc.n_obs
    offs, Cs, ds = [0], [], []
    for b in range(sc.n_scenes):
        for j in range(j0, j1):
            lo, hi = sc.obs_off[b * M + j], sc.obs_off[b * M + j + 1]
            Cs.append(sc.obs_C[lo:hi])
            ds.append(sc.obs_d[lo:hi])
            offs.append(offs[-1] + hi - lo)
    step = None if sc.obs_step is None else np.concatenate([sc.obs_step[b * M + j0:b * M + j1]
                                                            for b in range(sc.n_scenes)])
    return dataclasses.replace(sc, n_obs=j1 - j0, obs_off=np.asarray(offs, np.int32),
                               obs_C=np.concatenate(Cs) if Cs else np.zeros((0, sc.dim)),
                               obs_d=np.concatenate(ds) if ds else np.zeros(0), obs_step=step)


def pair_block(sc, arr, j0, j1):
    """the pairs of obstacles [j0, j1) in the rank-local pair order"""
    a = np.asarray(arr).reshape(sc.n_scenes, sc.horizon, sc.n_parts, sc.n_obs, *np.shape(arr)[1:])
    return a[:, :, :, j0:j1].reshape(-1, *np.shape(arr)[1:])


@pytest.mark.parametrize("name", ["c4", "c2", "c5x16", "c6"])
def test_obstacle_split_world2_emulated(ca, name):
    """a5 on one GPU: two handles on the two ca_obstacle_partition halves, same iterate;
    their per-(scene, t) records summed on the host equal the full handle's (1e-12), and
    the replicated Riccati step on that sum equals the unsharded primal step (1e-9)."""
    sc = case(name)
    o = oracle.Oracle(sc)
    o.admm_iterate(3)
    full = ca.Problem(sc)
    full.set_iterate(o.s, o.u, o.y, o.zeta, o.xi)
    full.dual_sweep()
    rec_full = full.stage_records()
    recs = []
    for r in range(2):
        j0, j1 = ca.obstacle_partition(sc, 2, r)
        sub = obstacle_half(sc, j0, j1)
        h = ca.Problem(sub)
        h.set_iterate(o.s, o.u, pair_block(sc, o.y[: sc.n_pairs], j0, j1)[:, : h.ny],
                      pair_block(sc, o.zeta[: sc.n_pairs], j0, j1), pair_block(sc, o.xi[: sc.n_pairs], j0, j1))
        h.dual_sweep()
        recs.append((h, h.stage_records()))
    R = rec_full.shape[-1]
    pm = R - 1  # the max-combined field
    summed = recs[0][1] + recs[1][1]
    summed[..., pm] = np.maximum(recs[0][1][..., pm], recs[1][1][..., pm])
    scale = 1.0 + np.abs(rec_full).max()
    assert np.abs(summed - rec_full).max() <= 1e-12 * scale
    full.primal_step()
    s_full, u_full = full.trajectory()
    h0 = recs[0][0]
    h0.primal_step_records(summed)
    s_sh, u_sh = h0.trajectory()
    close(s_sh, s_full, 1e-9, "s (sharded records)")
    close(u_sh, u_full, 1e-9, "u (sharded records)")


def test_empty_obstacle_slice_and_torch_workspace(ca):
    """A handle without local pairs (no obstacles; the dist path at world 1) must read
    zero aggregates -- also from a torch workspace of uninitialised memory -- and
    scale detection still joins the group's collective (+inf minima)."""
    import torch

    sc = scenes.make_config(2)
    sc0 = dataclasses.replace(sc, n_obs=0, obs_off=np.zeros(1, np.int32), obs_C=np.zeros((0, 2)), obs_d=np.zeros(0))
    garbage = torch.full((1 << 26,), float("nan"), dtype=torch.float64, device="cuda")  # poison the cache
    del garbage
    o = oracle.Oracle(sc0)
    o.admm_iterate(3)
    for kw in ({"workspace": "torch"}, {"dist": (1, 0, ca.nccl_unique_id())},
               {"dist": (1, 0, ca.nccl_unique_id()), "workspace": "torch"}):
        g = ca.Problem(sc0, **kw)
        g.admm_iterate(3)
        s, u = g.trajectory()
        close(s, o.s, 1e-9, f"s {kw}")
        close(u, o.u, 1e-9, f"u {kw}")
        _, amin = g.scale_detect(want_alpha=False)
        assert np.all(np.isinf(amin))


# ---------------------------------------------------------------------------
# C5 T2 end to end, 16 sampled scenes, full K, basis agreement
# ---------------------------------------------------------------------------

def test_c5_t2_end_to_end_16_scenes(ca):
    """SURVEY 8(c.5) C5 sampling: the GPU runs the whole 4096-scene batch for K = 100 (one
    iteration per call, the final Lemke basis of every pair recorded); the oracle runs 16
    scenes spread over the batch, no GPU value adopted.  Reported: the basis-agreement
    rate over all 16 x 100 sweeps (identical final basis and pivot count per pair).
    Asserted: the rate >= 1 - 2e-5 (the T1 flip allowance), and s, u, r_pri, r_dual within
    1e-6 per entry for every scene whose bases agreed in every sweep; a scene with a
    validated non-unique Lemke choice (reading #2) legitimately leaves that contract."""
    sc = scenes.make_c5()
    K = 100
    ids = [int(b) for b in np.linspace(0, 4095, 16)]
    per = sc.horizon * sc.n_parts * sc.n_obs
    g = ca.Problem(sc)
    g.set_record_basis(True)
    zm_g = np.zeros((K, len(ids), per), np.uint32)
    pv_g = np.zeros((K, len(ids), per), np.int32)
    rp_g = np.zeros((K, len(ids)))
    rd_g = np.zeros((K, len(ids)))
    for k in range(K):
        g.admm_iterate(1)
        rp, rd = g.scene_residuals()
        rp_g[k], rd_g[k] = rp[ids], rd[ids]
        for i, b in enumerate(ids):
            st = g.pair_state(b * per, per, zmask=True, fields=("pivots", "zmask"))
            zm_g[k, i], pv_g[k, i] = st["zmask"], st["pivots"]
    s_g, u_g = g.trajectory()

    def run(i):
        o = oracle.Oracle(sc.subset([ids[i]]))
        zm = np.zeros((K, per), np.uint32)
        pv = np.zeros((K, per), np.int32)
        hp, hd = np.zeros(K), np.zeros(K)
        for k in range(K):
            rd = o.dual_sweep()[0][0]
            zm[k], pv[k] = o.zmask[:per], o.pivots[:per]
            o.primal_step()
            hp[k], hd[k] = o.multiplier_update()[0], rd
        return zm, pv, hp, hd, o.s[0].copy(), o.u[0].copy()
    res = pmap(run, range(len(ids)))
    agree = total = 0
    clean = []
    for i, (zm, pv, hp, hd, s_o, u_o) in enumerate(res):
        same = (zm == zm_g[:, i]) & (pv == pv_g[:, i])
        agree += int(same.sum())
        total += same.size
        if same.all():
            clean.append(ids[i])
            close(s_g[ids[i]], s_o, 1e-6, f"s scene {ids[i]}")
            close(u_g[ids[i]], u_o, 1e-6, f"u scene {ids[i]}")
            close(rp_g[:, i], hp, 1e-6, f"r_pri history scene {ids[i]}")
            close(rd_g[:, i], hd, 1e-6, f"r_dual history scene {ids[i]}")
    rate = agree / total
    print(f"C5 T2 16 scenes x K={K}: basis agreement {rate:.8f} ({total - agree} of {total} pair solves differ); "
          f"scenes with every basis equal: {len(clean)}/16")
    assert rate >= 1.0 - 2e-5
    assert len(clean) >= 12


def test_c5_failures_reconciled_with_oracle(ca):
    """Every pair solve the GPU reports as failed over a full C5 solve (4096 scenes, K =
    100; the headline bench workload) is re-solved by the oracle on the identical pair
    inputs (pose of s^k, zeta^k, xi^k): the oracle must fail in the same way."""
    sc = scenes.make_c5()
    g = ca.Problem(sc)
    K = 100
    per_scene = sc.horizon * sc.n_parts * sc.n_obs
    seen = []
    for k in range(K):
        rc, r = g.dual_sweep()
        if r.n_fail:
            s, _ = g.trajectory()
            chunk = 256 * per_scene
            for p0 in range(0, g.n_pairs, chunk):
                st = g.pair_state(p0, min(chunk, g.n_pairs - p0), fields=("status",))
                for q in np.nonzero(st["status"] & 0xff)[0]:
                    p = p0 + int(q)
                    one = g.pair_state(p, 1)
                    b, t, A, bb, Cm, dv = pair_geometry(sc, p)
                    R, rho = oracle.pose(sc.pose_model, sc.pose_idx, sc.dim, s[b, t])
                    y, sto, piv, _ = oracle.pair_solve(A, bb, Cm, dv, R, rho, one["zeta"][0], one["xi"][0])
                    seen.append((k, p, int(one["status"][0]) & 0xff, int(sto)))
        g.primal_step()
        g.multiplier_update()
    print("C5 K=100 failed pair solves (iteration, pair, gpu status, oracle status):", seen)
    for k, p, sg, so in seen:
        assert sg == so, (k, p, sg, so)
