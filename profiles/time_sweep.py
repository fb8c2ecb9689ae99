"""Quick k_sweep timing on a C5 subset (CUDA events inside the library).

    python profiles/time_sweep.py [n_scenes] [iters]

Prints ms per fused k_sweep launch (iterations 2..K, after warm-up), mean pivots
and the Lemke failure count -- the loop used while tuning the sweep kernel.
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2406_07048_b200 as ca  # noqa: E402
import scenes  # noqa: E402

nsc = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 10
sc = scenes.make_c5(n_scenes=nsc)
g = ca.Problem(sc)
g.admm_iterate(3)  # warm-up
g.set_timing(True)
g.kernel_times(reset=True)
rc, h = g.admm_iterate(iters)
kt = g.kernel_times()
ms, nl = kt["sweep"]
print(f"scenes {nsc} iters {iters}: k_sweep {ms / nl:.3f} ms/launch  ({sc.n_pairs / (ms / nl) / 1e6:.1f} M pair/ms^-1... "
      f"{sc.n_pairs / (ms / nl * 1e-3) / 1e9:.3f} G pair-QP/s)  pivots/pair {h['pivots'].sum() / (iters * sc.n_pairs):.3f} "
      f"fail {int(h['n_fail'].sum())}  primal {kt['primal'][0] / max(1, kt['primal'][1]):.3f} ms")
