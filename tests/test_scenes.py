"""The seeded generators produce valid problems (SURVEY §8(d) recipe): unit-norm
rows, robot parts containing their body origin (b > 0), bounded nonempty
obstacles, reproducible seeds, C5 scenes regenerable one by one."""
import numpy as np
import pytest
from scipy.optimize import linprog

import scenes


@pytest.mark.parametrize("cfg", [1, 2, 3, 4])
def test_valid(cfg):
    sc = scenes.make_config(cfg)
    assert (sc.part_b > 0).all()
    np.testing.assert_allclose(np.linalg.norm(sc.part_A, axis=1), 1.0, rtol=1e-12)
    np.testing.assert_allclose(np.linalg.norm(sc.obs_C, axis=1), 1.0, rtol=1e-12)
    d = sc.dim
    for o in range(sc.n_scenes * sc.n_obs):
        Cm = sc.obs_C[sc.obs_off[o]:sc.obs_off[o + 1]]
        dv = sc.obs_d[sc.obs_off[o]:sc.obs_off[o + 1]]
        assert len(dv) >= d + 1
        for k in range(d):  # bounded: max/min of each coordinate finite
            for sgn in (1, -1):
                c = np.zeros(d)
                c[k] = -sgn
                r = linprog(c, A_ub=Cm, b_ub=dv, bounds=[(None, None)] * d, method="highs")
                assert r.status == 0
    assert sc.n_max <= 32


def test_reproducible_and_subset():
    a, b = scenes.make_config(2), scenes.make_config(2)
    assert np.array_equal(a.obs_C, b.obs_C) and np.array_equal(a.obs_d, b.obs_d)
    full = scenes.make_c5(n_scenes=6)
    sub = scenes.make_c5(scene_ids=[4, 1])
    assert np.array_equal(full.subset([4, 1]).obs_d, sub.obs_d)
    assert full.n_pairs == 6 * 50 * 200
    lo, hi = np.diff(full.obs_off).min(), np.diff(full.obs_off).max()
    assert lo >= 4 and hi <= 8
