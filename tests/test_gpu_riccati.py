"""The parallel-in-time primal step (k_riccati_scan) over horizons from the scan's
threshold (N = 8: 9 elements, 4 levels; partial last chunks of the forward rollout) to
horizons long enough that 4 (N + 1) threads exceed what the kernel's register count
allows in one CTA, so the kernel strides over the stages (ca_api.cu caps the CTA at
cudaFuncAttributes.maxThreadsPerBlock).  T1 primal step against the oracle at 1e-9."""
import numpy as np
import pytest

import oracle
import scenes

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ca():
    from paper_2406_07048_b200 import build

    build.build()
    import paper_2406_07048_b200 as ca

    return ca


def close(a, b, rtol, what):
    a, b = np.asarray(a), np.asarray(b)
    err = np.abs(a - b) / np.maximum(1.0, np.abs(b))
    assert err.max() <= rtol, f"{what}: max rel err {err.max():.3e}"


@pytest.mark.parametrize("N", [8, 9, 15, 16, 17, 33, 64, 90])
def test_scan_long_horizon_t1(ca, N):
    polys = [scenes.box_hrep([6.0, 0.5], [1.0, 1.0]), scenes.box_hrep([14.0, -0.6], [1.2, 0.8])]
    sc = scenes._car_common("C2L", 2, 7, N=N, iters=20, speed=8.0, polys_per_scene=[polys])
    o = oracle.Oracle(sc)
    o.admm_iterate(3)
    g = ca.Problem(sc)
    g.set_iterate(o.s, o.u, o.y, o.zeta, o.xi)
    o.set_iterate()
    g.dual_sweep()
    o.dual_sweep()
    g.primal_step()
    o.primal_step()
    s, u = g.trajectory()
    close(s, o.s, 1e-9, "s after primal step")
    close(u, o.u, 1e-9, "u after primal step")


def test_serial_recursion_path_still_matches_oracle():
    """The warp recursion (`k_riccati`) is what n_s > 4 and CA_RICCATI_SCAN=0 run; with the
    scan taking every small n_s <= 4 batch, run the T1 / T2 parity tests of those configs
    once more with the scan off (the switch is read once per process: a subprocess)."""
    import os
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, CA_RICCATI_SCAN="0")
    cmd = [sys.executable, "-m", "pytest", "-q", "-x", "-p", "no:cacheprovider", "-m", "gpu",
           os.path.join(root, "tests", "test_gpu_parity.py"), "-k",
           "t1_primal and (1 or 2 or 4 or 8) or t2_full and (2 or 4)"]
    out = subprocess.run(cmd, cwd=root, env=env, capture_output=True, text=True, timeout=900)
    assert out.returncode == 0, out.stdout[-3000:] + out.stderr[-2000:]
    assert " passed" in out.stdout
