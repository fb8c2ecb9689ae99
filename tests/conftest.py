import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) and the built CUDA library")
    config.addinivalue_line("markers", "slow: long-running CPU test")


@pytest.fixture(scope="session")
def orc():
    import oracle

    oracle.build()
    return oracle


# ----------------------------------------------------------------------------
# geometry helpers for the pins (test-only; independent of oracle/ and product)
# ----------------------------------------------------------------------------

def rot2(th):
    c, s = np.cos(th), np.sin(th)
    return np.array([[c, -s], [s, c]])


def poly_from_vertices(V):
    """H-rep (unit rows) of the convex polygon with CCW vertices V."""
    E = np.roll(V, -1, axis=0) - V
    N = np.stack([E[:, 1], -E[:, 0]], 1)
    N /= np.linalg.norm(N, axis=1, keepdims=True)
    return N, np.einsum("ij,ij->i", N, V)


def random_convex_polygon(rng, center, rmin=0.5, rmax=2.0, nmin=3, nmax=8):
    nv = int(rng.integers(nmin, nmax + 1))
    base = 2 * np.pi * np.arange(nv) / nv
    ang = base + rng.uniform(-0.2, 0.2, nv) * 2 * np.pi / nv + rng.uniform(0, 2 * np.pi)  # max gap < pi
    r = np.full(nv, rng.uniform(rmin, rmax))  # on a circle: convex in angle order
    V = np.asarray(center)[None] + r[:, None] * np.stack([np.cos(ang), np.sin(ang)], 1)
    return V


def sat_disjoint_2d(V1, V2, tol=0.0):
    """Separating-axis test for two convex polygons given by CCW vertices (textbook)."""
    for V in (V1, V2):
        E = np.roll(V, -1, axis=0) - V
        for e in E:
            n = np.array([e[1], -e[0]])
            p1, p2 = V1 @ n, V2 @ n
            if p1.max() < p2.min() - tol or p2.max() < p1.min() - tol:
                return True
    return False
