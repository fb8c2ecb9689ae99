"""Probe (CPU, oracle only): can a pair LCP's answer be certified from the previous
ADMM iteration's support instead of re-running Lemke (a warm start that is exact only
where the LCP solution is unique)?  For a monotone LCP, uniqueness follows from strict
complementarity at z plus a nonsingular M_aa.  This samples C5 pairs after 20 ADMM
iterations and reports the support size, whether w > 0 off the support, and the
conditioning of M_aa.

    python profiles/warm_certificate_probe.py  > profiles/r02/warm_certificate_probe.txt

Finding (round 2): ~every pair ends with w = 0 on ALL of y_U (u* = K^T y + b = 0: the
QP's minimiser set is a whole face, Lemke returns one vertex of it), so no pair is
strictly complementary -- the answer depends on Lemke's pivot path, and a support
warm start cannot reproduce it.  (The prox variant, reading #2, has a unique minimiser
and IS warm-started: NEXT f4.)
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import oracle  # noqa: E402
import scenes  # noqa: E402
from parity_util import pair_geometry  # noqa: E402

sc = scenes.make_c5(scene_ids=[0, 1000])
o = oracle.Oracle(sc)
o.admm_iterate(20)
s, zeta, xi = o.s.copy(), o.zeta.copy(), o.xi.copy()
rng = np.random.default_rng(0)
stats = {}
nzero_w = []
for p in rng.choice(sc.n_pairs, 400, replace=False):
    b, t, A, bb, Cm, dv = pair_geometry(sc, p)
    R, rho = oracle.pose(sc.pose_model, sc.pose_idx, sc.dim, s[b, t])
    K, bvec, e, M, q = oracle.pair_lcp(A, bb, Cm, dv, R, rho, zeta[p], xi[p])
    z, st, piv, basis = oracle.lemke(M, q)
    w = M @ z + q
    al = z > 1e-12
    scale = 1 + np.abs(q).max()
    strict = bool(np.all(w[~al] > 1e-9 * scale))
    cond = np.linalg.cond(M[np.ix_(al, al)]) if al.any() else 0.0
    nzero_w.append(int(np.sum(np.abs(w[~al]) <= 1e-9 * scale)))
    key = (int(al.sum()), strict, bool(cond < 1e8))
    stats[key] = stats.get(key, 0) + 1
print("C5 scenes 0, 1000 after 20 ADMM iterations, 400 sampled pairs")
print("(support size, strictly complementary, cond(M_aa) < 1e8): count")
for k, v in sorted(stats.items()):
    print(k, v)
print("mean count of w_i = 0 off the support (degenerate rows):", float(np.mean(nzero_w)))
