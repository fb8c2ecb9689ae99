"""Subprocess body of tests/test_gpu_checked.py: runs a fixed set of problems through
the library CA_LIBRARY points at and saves every output to an .npz (bitwise compare)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import dataclasses  # noqa: E402

import numpy as np  # noqa: E402

import paper_2406_07048_b200 as ca  # noqa: E402
import scenes  # noqa: E402
from test_gpu_parity import many_faced_scene, symmetric_scene  # noqa: E402


def cases():
    c2 = scenes.make_config(2)
    yield "c1", scenes.make_config(1), {}, 10
    yield "c2", c2, {}, 10
    yield "c3", scenes.make_config(3), {}, 5
    yield "c4", scenes.make_config(4), {}, 5
    yield "c2b", scenes.make_config(8), {}, 10
    yield "c2t", scenes.make_config(10), {}, 10
    yield "c4s", scenes.make_config(9), {}, 5
    yield "c2n", scenes.make_config(7), {}, 5
    yield "c11", scenes.make_config(11), {}, 5
    yield "c12", scenes.make_config(12), {}, 5
    yield "c2prox", c2, {"prox_eps": 1e-2}, 5
    yield "c2proxlemke", c2, {"prox_eps": 1e-2, "prox_solver": 1}, 3
    yield "c5x64", scenes.make_c5(n_scenes=64), {}, 3
    yield "c5x64prox", scenes.make_c5(n_scenes=64), {"prox_eps": 1e-2}, 3
    yield "c5x1100", scenes.make_c5(n_scenes=1100), {}, 2
    yield "sym", symmetric_scene(), {}, 5
    yield "largen", many_faced_scene(), {}, 5
    yield "zero", dataclasses.replace(c2, n_obs=0, obs_off=np.zeros(1, np.int32), obs_C=np.zeros((0, 2)),
                                      obs_d=np.zeros(0)), {}, 3


def main(out):
    res = {}
    for name, sc, kw, K in cases():
        g = ca.Problem(sc, **kw)
        g.scale_detect()
        rc, h = g.admm_iterate(K)
        s, u = g.trajectory()
        st = g.pair_state(0, min(g.n_pairs, 50000)) if g.n_pairs else {}
        a, amin = g.scale_detect()
        res[name + "_s"], res[name + "_u"] = s, u
        res[name + "_rpri"], res[name + "_piv"] = h["r_pri"], h["pivots"]
        res[name + "_amin"] = amin
        for k, v in st.items():
            res[f"{name}_{k}"] = v
        if name == "c2":
            g2 = ca.Problem(sc, eps_pri=0.2, eps_dual=0.2, max_iters=60)
            rc, rep, it, cv = g2.admm_solve()
            res["solve_it"], res["solve_s"] = it, g2.trajectory()[0]
        g.close()
    np.savez(out, **res)
    print("checked_run ok", len(res))


if __name__ == "__main__":
    main(sys.argv[1])
