"""Wall-clock per ca_admm_iterate(K) solve of a configuration (timing events off, so
the CUDA-graph path is used), min over repeats.

    python profiles/time_solve.py <config> [repeats]
"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2406_07048_b200 as ca  # noqa: E402
import scenes  # noqa: E402

cfg = int(sys.argv[1])
rep = int(sys.argv[2]) if len(sys.argv) > 2 else 5
sc = scenes.make_config(cfg)
g = ca.Problem(sc)
K = sc.iters
best = 1e9
for r in range(rep + 1):
    g.reset_iterate()
    t0 = time.perf_counter()
    g.admm_iterate(K, hist=False)
    dt = time.perf_counter() - t0
    if r:
        best = min(best, dt)
print(f"config {cfg}: K={K} {best * 1e3:.2f} ms per solve ({best / K * 1e6:.1f} us/iteration, "
      f"{sc.n_pairs * K / best / 1e6:.2f} M pair-QP/s)")
