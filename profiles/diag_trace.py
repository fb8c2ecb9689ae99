"""Trace the GPU Lemke path of the first failing C5 pair (diagnostics)."""
import os, sys, pickle
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import oracle, scenes, paper_2406_07048_b200 as ca
from parity_util import pair_geometry
sc = scenes.make_c5(n_scenes=512)
g = ca.Problem(sc)
out = []
for it in range(40):
    s, u = g.trajectory(); st0 = g.pair_state()
    rc, r = g.dual_sweep()
    st1 = g.pair_state()
    bad = np.nonzero(st1["status"] != 0)[0]
    if len(bad):
        for p in bad[:3]:
            g.set_iterate(y=st0["y"])
            g.debug_trace(int(p))
            g.dual_sweep()
            tr = g.debug_trace(-1)
            b, t, A, bb, Cm, dv = pair_geometry(sc, p)
            R, rho = oracle.pose(1, [0, 1, 2], 2, s[b, t])
            out.append(dict(A=A, bb=bb, Cm=Cm, dv=dv, R=R, rho=rho, zeta=st0["zeta"][p], xi=st0["xi"][p], trace=tr,
                            gpu_piv=st1["pivots"][p]))
        break
    g.primal_step(); g.multiplier_update()
os.makedirs("gpurun_out", exist_ok=True)
pickle.dump(out, open("gpurun_out/fail_trace.pkl", "wb"))
print("dumped", len(out))
