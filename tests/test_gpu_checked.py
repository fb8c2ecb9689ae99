"""T4 of SURVEY §4 without compute-sanitizer (closed on this pool: runs under it left
GPUs needing a reset).  Substitutes, each on the product kernels:
  memcheck   -> a checked build (-DCA_CHECKED): device-side bounds / layout assertions
                on every index the per-pair kernels derive and on each kernel's dynamic
                shared-memory extent; a failure traps (CA_E_CUDA).  It must run a wide
                set of problems cleanly and give BITWISE the product library's results.
  initcheck  -> every buffer carved out of a NaN-poisoned torch workspace: results
                bitwise those of a fresh cudaMalloc'd handle.
  racecheck  -> the persistent sweep re-run with a capped grid (CA_SWEEP_WARPS: another
                item-to-warp interleaving and timing) and run twice: bitwise identical
                (no FP atomics, one writer per record slot).
"""
import os
import subprocess
import sys

import numpy as np
import pytest

import scenes

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHECKED = os.path.join(ROOT, "scratch", "libs", "checked.so")


@pytest.fixture(scope="module")
def ca():
    from paper_2406_07048_b200 import build

    build.build()
    import paper_2406_07048_b200 as ca

    return ca


def run_lib(lib, out, env_extra=None):
    env = dict(os.environ, **(env_extra or {}))
    if lib:
        env["CA_LIBRARY"] = lib
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tests", "checked_run.py"), out], env=env,
                       capture_output=True, text=True, timeout=1500)
    assert r.returncode == 0, (r.stdout[-2000:], r.stderr[-3000:])
    return np.load(out)


def assert_same(a, b):
    assert set(a.files) == set(b.files)
    bad = [k for k in a.files if not np.array_equal(a[k], b[k], equal_nan=True)]
    assert not bad, bad


def test_checked_build_bitwise(ca, tmp_path):
    if not os.path.exists(CHECKED):
        from paper_2406_07048_b200 import build

        build.build(out=CHECKED, defines=("CA_CHECKED",))
    prod = run_lib(None, str(tmp_path / "prod.npz"))
    chk = run_lib(CHECKED, str(tmp_path / "checked.npz"))
    assert_same(prod, chk)


def test_capped_grid_and_rerun_bitwise(ca, tmp_path):
    a = run_lib(None, str(tmp_path / "a.npz"))
    b = run_lib(None, str(tmp_path / "b.npz"), {"CA_SWEEP_WARPS": "148"})
    c = run_lib(None, str(tmp_path / "c.npz"), {"CA_SWEEP_WARPS": "37"})
    assert_same(a, b)
    assert_same(a, c)


@pytest.mark.parametrize("cfg,n", [(2, None), (4, None), (8, None), (5, 64), (5, 1100)])
def test_poisoned_workspace_bitwise(ca, cfg, n):
    import torch

    sc = scenes.make_c5(n_scenes=n) if cfg == 5 else scenes.make_config(cfg)
    ref = ca.Problem(sc)
    ref.admm_iterate(4)
    s0, u0 = ref.trajectory()
    st0 = ref.pair_state(0, min(ref.n_pairs, 20000))
    ref.close()
    poison = torch.full((1 << 28,), float("nan"), dtype=torch.float64, device="cuda")  # 2 GiB of NaN
    del poison  # the caching allocator hands this memory to the workspace below
    g = ca.Problem(sc, workspace="torch")
    g.admm_iterate(4)
    s1, u1 = g.trajectory()
    st1 = g.pair_state(0, min(g.n_pairs, 20000))
    assert np.array_equal(s0, s1) and np.array_equal(u0, u1)
    for k in st0:
        assert np.array_equal(st0[k], st1[k]), k
