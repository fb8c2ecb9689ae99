"""Run one configuration for ncu captures of the small-config kernels.

    python profiles/prof_cfg.py <config 1-5> [iters] [n_scenes (C5)]
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2406_07048_b200 as ca  # noqa: E402
import scenes  # noqa: E402

cfg = int(sys.argv[1])
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 5
kw = {"n_scenes": int(sys.argv[3])} if len(sys.argv) > 3 else {}
sc = scenes.make_config(cfg, **kw)
g = ca.Problem(sc)
g.set_timing(True)
rc, h = g.admm_iterate(iters)
kt = g.kernel_times()
print("ok", cfg, iters, {k: (round(v[0] / max(1, v[1]), 4), v[1]) for k, v in kt.items()})
