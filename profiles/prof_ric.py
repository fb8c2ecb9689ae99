"""Driver for ncu captures of the small-batch primal-step kernel: C4 replicated over
n scenes (64 by default: enough CTAs for stall sampling, still the small-batch path)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2406_07048_b200 as ca  # noqa: E402
import scenes  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 64
sc = scenes.make_config(4).subset([0] * n)
g = ca.Problem(sc)
g.admm_iterate(4)
print("ok")
