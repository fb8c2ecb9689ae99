"""bench.py's multi-GPU code paths at one GPU (the driver's N>1 runs are the first
time they see more ranks): --force-dist runs the scene-sharded mode (NCCL
communicator of one rank, per-iteration scene-statistics exchange forced on with
CA_FORCE_SCENE_GRID) and the obstacle-sharded mode, each on a small C5 batch, and
checks that the JSON line is complete and its pivots / failures agree with the
plain single-GPU run on the same scenes.
"""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def run_bench(*extra):
    cmd = [sys.executable, os.path.join(ROOT, "bench.py"), "--steps", "3", "--warmup", "3", "--scenes", "128",
           "--no-cpu", "--e2e-steps", "1", *extra]
    env = {k: v for k, v in os.environ.items() if k not in ("RANK", "WORLD_SIZE", "LOCAL_RANK")}
    out = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-3000:]
    line = [x for x in out.stdout.splitlines() if x.startswith("{")][-1]
    return json.loads(line)


@pytest.mark.parametrize("shard", ["scenes", "obstacles"])
def test_bench_dist_modes_at_one_gpu(shard):
    plain = run_bench()
    d = run_bench("--shard", shard, "--force-dist")
    for k in ("metric", "value", "unit", "roofline", "e2e", "gpu_launches", "clocks", "config"):
        assert k in d, k
    assert d["value"] > 0 and d["e2e"]["value"] > 0 and d["gpu_launches"] > 0
    assert d["n_gpus"] == 1 and d["config"].get("force_dist") is True
    assert d["nccl_collectives"] > 0 and plain["nccl_collectives"] == 0
    # the same scenes and iterations: identical work
    assert d["lemke_failure_kinds"] == plain["lemke_failure_kinds"]
    assert d["max_pivots"] == plain["max_pivots"]
