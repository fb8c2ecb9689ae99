"""Diagnose Lemke failures on C5: GPU statuses vs the oracle on identical pair inputs."""
import os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import oracle, scenes, paper_2406_07048_b200 as ca
from parity_util import pair_geometry
nsc = int(sys.argv[1]) if len(sys.argv) > 1 else 256
sc = scenes.make_c5(n_scenes=nsc)
g = ca.Problem(sc)
tot = {}
dumps = []
for it in range(40):
    s, u = g.trajectory(); st0 = g.pair_state()
    rc, r = g.dual_sweep()
    st1 = g.pair_state()
    bad = np.nonzero((st1["status"] & 0xff) != 0)[0]
    tot["fallback"] = tot.get("fallback", 0) + int(((st1["status"] & 0x100) != 0).sum())
    for p in bad[:20]:
        b, t, A, bb, Cm, dv = pair_geometry(sc, p)
        R, rho = oracle.pose(1, [0, 1, 2], 2, s[b, t])
        y, sto, piv, basis = oracle.pair_solve(A, bb, Cm, dv, R, rho, st0["zeta"][p], st0["xi"][p])
        dumps.append(dict(A=A, bb=bb, Cm=Cm, dv=dv, R=R, rho=rho, zeta=st0["zeta"][p], xi=st0["xi"][p],
                          gpu_piv=st1["pivots"][p], gpu_y=st1["y"][p]))
        key = (int(st1["status"][p]), int(sto))
        tot[key] = tot.get(key, 0) + 1
        if tot[key] <= 3:
            print("iter", it, "pair", p, "gpu status", st1["status"][p], "gpu piv", st1["pivots"][p], "| oracle status", sto, "piv", piv, "n", len(y))
    g.primal_step(); g.multiplier_update()
print("counts (gpu_status, oracle_status):", tot)
import pickle; os.makedirs("gpurun_out", exist_ok=True); pickle.dump(dumps, open("gpurun_out/fail_pairs.pkl", "wb"))
