"""Host logic of the receding-horizon driver (no GPU: the oracle backend)."""
import numpy as np

import scenes
from paper_2406_07048_b200 import mpc
from parity_util import OracleSolver


def test_shift_pairs_moves_timesteps():
    sc = scenes.make_config(2)
    G = sc.n_parts * sc.n_obs
    t_of = np.repeat(np.arange(sc.horizon), G).astype(float)  # value = timestep index
    sh = mpc.shift_pairs(t_of, sc).reshape(sc.horizon, G)
    assert np.array_equal(sh[:-1, 0], np.arange(1, sc.horizon))
    assert np.all(sh[-1] == sc.horizon - 1)


def test_unicycle_step_is_the_linearised_model_at_zero_input():
    s = np.array([1.0, 2.0, 0.3, 5.0])
    A, B, c = scenes.unicycle_ltv(s[None])
    assert np.allclose(mpc.unicycle_step(s, np.zeros(2)), A[0] @ s + c[0], atol=1e-14)


def test_oracle_closed_loop_advances():
    sc = scenes.make_config(2)
    loop = mpc.RecedingHorizon(sc, K=15, speed=3.0, solver=OracleSolver())
    x0 = loop.s_now[0]
    for _ in range(3):
        loop.step()
    assert loop.s_now[0] > x0 + 0.5  # ~3 m/s for 0.3 s
    s_sol = loop.prev[0]
    assert s_sol.shape == (sc.horizon + 1, sc.n_state)
