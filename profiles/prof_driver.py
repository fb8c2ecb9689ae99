"""Small driver for ncu captures of the hot kernels (C5 subset, same launch shape).

    python profiles/prof_driver.py [n_scenes] [iters]
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2406_07048_b200 as ca  # noqa: E402
import scenes  # noqa: E402

nsc = int(sys.argv[1]) if len(sys.argv) > 1 else 256
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 4
sc = scenes.make_c5(n_scenes=nsc)
g = ca.Problem(sc)
g.scale_detect(want_alpha=False)
rc, h = g.admm_iterate(iters)
g.scale_detect(want_alpha=False)
print("ok", nsc, iters, h["pivots"].mean() / sc.n_pairs, h["n_fail"].sum())
