"""Bitwise A/B of two library builds on the same problem: trajectory, per-scene residuals and
the per-pair state after K iterations must be identical (a change that only reorders or
restages work).   CA_LIBRARY=<lib> python profiles/bitwise_ab.py <out.npz> [cfg] [scenes] [K]"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2406_07048_b200 as ca  # noqa: E402
import scenes  # noqa: E402

out = sys.argv[1]
cfg = int(sys.argv[2]) if len(sys.argv) > 2 else 5
nsc = int(sys.argv[3]) if len(sys.argv) > 3 else 64
K = int(sys.argv[4]) if len(sys.argv) > 4 else 5
sc = scenes.make_c5(n_scenes=nsc) if cfg == 5 else scenes.make_config(cfg)
g = ca.Problem(sc)
rc, h = g.admm_iterate(K)
s, u = g.trajectory()
rp, rd = g.scene_residuals()
st = g.pair_state(fields=("y", "zeta", "xi", "pivots"))
np.savez(out, s=s, u=u, rp=rp, rd=rd, y=st["y"], zeta=st["zeta"], xi=st["xi"], piv=st["pivots"],
         hist=np.array([h[f] for f in ("r_pri", "r_dual", "pivots")]))
print("saved", out)
