"""Per-step latency of the receding-horizon closed loop on the GPU (NEXT f2) against
the paper's 0.1 s control period.

    python profiles/closed_loop.py [steps]
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import scenes  # noqa: E402
from paper_2406_07048_b200 import mpc  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 30
for cfg, speed, name in ((2, 3.0, "C2 (4 obstacles, N=50, K=200)"), (6, 20.0, "C4m (100 moving vehicles, N=60, K=300)"),
                         (1, 8.0, "C1 (N=10, K=50)")):
    sc = scenes.make_config(cfg)
    loop = mpc.RecedingHorizon(sc, K=sc.iters, speed=speed)
    for _ in range(steps):
        loop.step()
    lat = np.array(loop.latency[1:]) * 1e3  # skip the first (handle creation)
    print(f"{name}: per MPC step median {np.median(lat):.2f} ms, max {lat.max():.2f} ms over {len(lat)} steps "
          f"(0.1 s period: {100 * np.median(lat) / 100:.1f} % used); x advanced {loop.s_now[0] - sc.s0[0, 0]:.1f} m")
