"""Receding-horizon closed loop (paper_2406_07048_b200/mpc.py): the
same driver with the GPU and with the CPU oracle as the solver -- warm-started
shifted iterates, per-step relinearisation, moving obstacles -- must produce the same
closed-loop trajectory."""
import dataclasses

import numpy as np
import pytest

import scenes
from paper_2406_07048_b200 import mpc
from parity_util import OracleSolver


def c4m_short():
    sc = scenes.make_config(6)
    keep = list(range(40))
    offs, Cs, ds = [0], [], []
    for j in keep:
        lo, hi = sc.obs_off[j], sc.obs_off[j + 1]
        Cs.append(sc.obs_C[lo:hi])
        ds.append(sc.obs_d[lo:hi])
        offs.append(offs[-1] + hi - lo)
    N = 30
    return dataclasses.replace(sc, n_obs=len(keep), horizon=N, obs_off=np.asarray(offs, np.int32),
                               obs_C=np.concatenate(Cs), obs_d=np.concatenate(ds),
                               obs_step=np.ascontiguousarray(sc.obs_step[keep]), dyn_A=sc.dyn_A[:N],
                               dyn_B=sc.dyn_B[:N], dyn_c=sc.dyn_c[:N], s_ref=sc.s_ref[:, :N + 1])


@pytest.mark.gpu
@pytest.mark.parametrize("case", ["c2", "c4m", "c2n", "c2b", "c4s"])
def test_closed_loop_gpu_equals_oracle(case):
    """c2n: the unicycle relinearised at every ADMM iterate inside each MPC solve;
    c2b: state/control boxes (NEXT f1), the plant saturating the applied control;
    c4s: sensing (NEXT f3) re-evaluated at every step as the ego advances."""
    sc, K, speed, steps = {"c2": (scenes.make_config(2), 40, 3.0, 5), "c4m": (c4m_short(), 30, 20.0, 3),
                           "c2n": (scenes.make_config(7), 40, 3.0, 5), "c2b": (scenes.make_config(8), 40, 3.0, 5),
                           "c4s": (dataclasses.replace(c4m_short(), sense_half=np.array([40.0, 8.0])), 30, 20.0, 3)}[case]
    runs = {}
    for backend in ("gpu", "oracle"):
        loop = mpc.RecedingHorizon(sc, K=K, speed=speed, solver=None if backend == "gpu" else OracleSolver())
        states, ctrls = [loop.s_now.copy()], []
        for _ in range(steps):
            ctrls.append(loop.step())
            states.append(loop.s_now.copy())
        runs[backend] = (np.array(states), np.array(ctrls), loop.prev[0])
    (sg, ug, tg), (so, uo, to) = runs["gpu"], runs["oracle"]
    scale = 1.0 + np.abs(so).max()
    assert np.abs(sg - so).max() <= 1e-6 * scale
    assert np.abs(ug - uo).max() <= 1e-6 * (1.0 + np.abs(uo).max())
    assert np.abs(tg - to).max() <= 1e-6 * (1.0 + np.abs(to).max())
