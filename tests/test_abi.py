"""CPU-side checks of the C-ABI boundary: the library loads, exports every symbol
include/ca.h declares, validates inputs before touching the GPU, and fails loudly
(CA_E_CUDA) where there is no B200 -- no CPU fallback."""
import dataclasses
import os
import re
import subprocess

import numpy as np
import pytest

import scenes

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "ca.h")


@pytest.fixture(scope="module")
def ca():
    from paper_2406_07048_b200 import build

    build.build()
    import paper_2406_07048_b200 as ca

    return ca


def header_symbols():
    txt = open(HEADER).read()
    return sorted(set(re.findall(r"\b(ca_[a-z0-9_]+)\s*\(", txt)))


def test_exports_every_header_symbol(ca):
    syms = header_symbols()
    assert len(syms) >= 18
    out = subprocess.run(["nm", "-D", "--defined-only", ca.library_path()], capture_output=True, text=True).stdout
    exported = set(re.findall(r" T (ca_[a-z0-9_]+)$", out, re.M))
    missing = [s for s in syms if s not in exported]
    assert not missing, missing
    L = ca.lib()
    for s in syms:
        assert hasattr(L, s)


def test_no_dynamic_cudart_dependency(ca):
    out = subprocess.run(["ldd", ca.library_path()], capture_output=True, text=True).stdout
    assert "libcudart" not in out


def _create(ca, sc, **kw):
    try:
        ca.Problem(sc, **kw)
    except ca.CAError as e:
        return e.code, str(e)
    return 0, ""


def test_validation_errors_precede_device(ca):
    sc = scenes.make_config(2)
    bad = dataclasses.replace(sc, part_b=-sc.part_b)
    assert _create(ca, bad)[0] == -3  # CA_E_GEOMETRY: b_i must be > 0 (reading #22)
    bad = dataclasses.replace(sc, dim=4)
    assert _create(ca, bad)[0] == -2  # CA_E_DIM
    assert _create(ca, sc, prox_eps=-1e-3)[0] == -1  # CA_E_INVALID (prox_eps >= 0, reading #2)
    assert _create(ca, sc, prox_eps=1e-2, prox_solver=2)[0] == -1  # CA_E_INVALID (NEXT f4: 0 or 1)
    assert _create(ca, dataclasses.replace(sc, pose_model=7))[0] == -4  # CA_E_UNSUPPORTED
    bad = dataclasses.replace(sc, Qs=-sc.Qs)
    assert _create(ca, bad)[0] == -1  # CA_E_INVALID (not SPD)
    step = np.zeros((sc.n_scenes * sc.n_obs, sc.dim))
    step[0, 0] = np.nan
    bad = dataclasses.replace(sc, obs_step=step)
    assert _create(ca, bad)[0] == -1  # CA_E_INVALID (moving obstacles: finite steps)
    c2b = scenes.make_config(8)  # boxes (NEXT f1): min <= max, no NaN, box_rho > 0
    assert _create(ca, dataclasses.replace(c2b, box_rho=0.0))[0] == -1
    assert _create(ca, dataclasses.replace(c2b, u_min=np.array([1.0, -1.0])))[0] == -1
    assert _create(ca, dataclasses.replace(c2b, s_max=np.array([np.nan, 1, 1, 1])))[0] == -1
    c2t = scenes.make_config(10)  # scaling centres (NEXT f3): the trailer needs its own
    assert _create(ca, dataclasses.replace(c2t, part_ctr=None))[0] == -3
    assert _create(ca, dataclasses.replace(c2t, part_ctr=np.array([[0.0, 0.0], [3.0, 0.0]])))[0] == -3


@pytest.mark.skipif(os.path.exists("/dev/nvidia0"), reason="GPU present")
def test_fails_loudly_without_gpu(ca):
    code, msg = _create(ca, scenes.make_config(1))
    assert code == -5 and "no CPU fallback" in msg


def test_obstacle_partition_properties(ca):
    """ca_obstacle_partition (host only): contiguous, disjoint, covering, face-balanced."""
    for cfg, kw in ((4, {}), (2, {}), (5, {"n_scenes": 3})):
        sc = scenes.make_config(cfg, **kw)
        faces = np.diff(sc.obs_off).reshape(sc.n_scenes, sc.n_obs).sum(0)
        for W in (1, 2, 3, 5, 8):
            parts = [ca.obstacle_partition(sc, W, r) for r in range(W)]
            assert parts[0][0] == 0 and parts[-1][1] == sc.n_obs
            for (a0, a1), (b0, b1) in zip(parts, parts[1:]):
                assert a1 == b0 and a0 <= a1
            tot = faces.sum()
            for r, (j0, j1) in enumerate(parts):
                got = faces[j0:j1].sum()
                assert abs(got - tot / W) <= faces.max() + 1e-9, (cfg, W, r, got, tot / W)


def test_workspace_size_host_only(ca):
    """ca_workspace_size is a host planning pass: positive, grows with the batch, and
    covers at least the pair state (y, zeta, xi, status) of every pair."""
    import ctypes as C

    from paper_2406_07048_b200._ca import make_desc

    def size(sc):
        keep = {}
        desc = make_desc(sc, keep)
        nb = C.c_size_t()
        rc = ca.lib().ca_workspace_size(C.byref(desc), None, C.byref(nb))
        assert rc == 0
        return nb.value

    small, big = scenes.make_c5(n_scenes=2), scenes.make_c5(n_scenes=8)
    s2, s8 = size(small), size(big)
    assert 0 < s2 < s8
    per_pair = 8 * (big.n_max + 1 + big.dim) + 4
    assert s8 >= big.n_pairs * per_pair
