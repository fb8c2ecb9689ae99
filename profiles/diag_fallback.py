"""Count dense-fallback re-solves (status bit 0x100) per sweep for a configuration.

    python profiles/diag_fallback.py <config> [iters] [n_scenes]
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2406_07048_b200 as ca  # noqa: E402
import scenes  # noqa: E402

cfg = int(sys.argv[1])
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 30
kw = {"n_scenes": int(sys.argv[3])} if len(sys.argv) > 3 else {}
sc = scenes.make_config(cfg, **kw)
g = ca.Problem(sc)
tot = 0
per = []
for k in range(iters):
    g.admm_iterate(1)
    st = g.pair_state()["status"]
    f = int(np.count_nonzero(st & 0x100))
    per.append(f)
    tot += f
print(f"config {cfg}: pairs/sweep {sc.n_pairs}, dense re-solves per sweep {np.mean(per):.2f} "
      f"(max {max(per)}), sweeps with any {sum(1 for x in per if x)}/{iters}")
