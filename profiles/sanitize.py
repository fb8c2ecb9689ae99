"""Sanitizer driver (SURVEY §4 tier T4): small runs of every kernel family through the
C ABI, meant to be executed under compute-sanitizer (memcheck / racecheck / synccheck /
initcheck), one tool per process:

    compute-sanitizer --tool racecheck python profiles/sanitize.py c2
    compute-sanitizer --tool racecheck python profiles/sanitize.py c5 64

c2  = C2 (one-wave latency mode: warp-cooperative dense Lemke, warp-per-scene Riccati),
      plus C3 (d = 3 scale detection, 7-state Riccati) and C2b (box block);
c5  = an n-scene C5 subset (persistent-warp revised Lemke with the dense fallback,
      pooled sort, thread-per-scene Riccati when n > 1024, grouped stage kernel).
Exits 0 after printing a one-line summary; the sanitizer's own report decides.
No torch import: device memory comes from the library's own cudaMalloc.
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import paper_2406_07048_b200 as ca  # noqa: E402
import scenes  # noqa: E402


def run(sc, iters, **kw):
    g = ca.Problem(sc, **kw)
    g.scale_detect()
    rc, h = g.admm_iterate(iters)
    g.dual_sweep()
    g.primal_step()
    g.multiplier_update()
    s, u = g.trajectory()
    g.pair_state(0, min(g.n_pairs, 1000))
    g.close()
    assert np.all(np.isfinite(s)) and np.all(np.isfinite(u))
    return h


def main():
    what = sys.argv[1] if len(sys.argv) > 1 else "c2"
    if what == "c2":
        h = run(scenes.make_config(2), 3)
        run(scenes.make_config(3), 2)
        run(scenes.make_config(8), 2)
        run(scenes.make_config(2), 2, prox_eps=1e-2)  # NEXT f4 dual Newton
    else:
        n = int(sys.argv[2]) if len(sys.argv) > 2 else 64
        h = run(scenes.make_c5(n_scenes=n), 2)
    print(f"sanitize {what}: ok, last r_pri {h['r_pri'][-1]:.3e} pivots {int(h['pivots'][-1])}", flush=True)


if __name__ == "__main__":
    main()
