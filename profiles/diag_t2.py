"""C5 end-to-end divergence diagnosis: GPU (full 4096-scene batch, one iteration per
call) vs the oracle on sampled scenes.  Per scene: the first iteration whose Lemke bases
differ, how many pairs differ there, how far apart the inputs of that sweep (s^k, zeta,
xi) already were, and the final trajectory error."""
import os
import sys
from concurrent.futures import ThreadPoolExecutor

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np  # noqa: E402

import oracle  # noqa: E402
import paper_2406_07048_b200 as ca  # noqa: E402
import scenes  # noqa: E402
from parity_util import validate_pair_choice  # noqa: E402

K = int(sys.argv[1]) if len(sys.argv) > 1 else 100
nb = int(sys.argv[2]) if len(sys.argv) > 2 else 16
full = len(sys.argv) > 3 and sys.argv[3] == "full"
sc = scenes.make_c5() if full else scenes.make_c5(n_scenes=max(nb, 64))
ids = [int(b) for b in np.linspace(0, sc.n_scenes - 1, nb)]
per = sc.horizon * sc.n_parts * sc.n_obs
g = ca.Problem(sc)
g.set_record_basis(True)
G = {b: [] for b in ids}
for k in range(K):
    s_pre, u_pre = g.trajectory()
    pre = {b: g.pair_state(b * per, per, fields=("y", "zeta", "xi")) for b in ids}
    g.admm_iterate(1)
    for b in ids:
        st = g.pair_state(b * per, per, zmask=True, fields=("pivots", "zmask", "y"))
        G[b].append((s_pre[b].copy(), pre[b], st))
s_fin, _ = g.trajectory()


def run(b):
    o = oracle.Oracle(sc.subset([b]))
    first = None
    for k in range(K):
        s_g, pre, st = G[b][k]
        ds = np.abs(o.s[0] - s_g).max() / max(1, np.abs(s_g).max())
        dz = np.abs(o.zeta[:per] - pre["zeta"]).max() / max(1, np.abs(pre["zeta"]).max())
        zeta_in, xi_in, s_in = o.zeta[:per].copy(), o.xi[:per].copy(), o.s.copy()
        o.dual_sweep()
        diff = np.nonzero((o.zmask[:per] != st["zmask"]) | (o.pivots[:per] != st["pivots"]))[0]
        if len(diff) and first is None:
            ok = 0
            for p in diff[:20]:
                try:
                    validate_pair_choice(sc.subset([b]), s_in, zeta_in, xi_in, p, st["y"][p], o.y[p])
                    ok += 1
                except AssertionError:
                    pass
            first = (k, len(diff), ds, dz, ok, min(20, len(diff)))
        o.primal_step()
        o.multiplier_update()
    err = np.abs(o.s[0] - s_fin[b]).max() / max(1, np.abs(o.s[0]).max())
    return b, first, err


with ThreadPoolExecutor(os.cpu_count()) as ex:
    for b, first, err in ex.map(run, ids):
        if first is None:
            print(f"scene {b}: bases equal in all {K} sweeps; final s rel err {err:.2e}")
        else:
            k, n, ds, dz, ok, nv = first
            print(f"scene {b}: first basis difference at iteration {k}: {n} pairs; inputs there differ by "
                  f"s {ds:.2e} zeta {dz:.2e}; {ok}/{nv} validated optimal; final s rel err {err:.2e}")
