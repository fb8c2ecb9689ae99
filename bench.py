#!/usr/bin/env python
"""Benchmark of the ADMM hot path of arXiv 2406.07048 on B200 (sm_100a, FP64).

One *step* = one full ADMM solve of the whole hot path over one batch (SURVEY
§8(a)): reset to the initial iterate (O1), scale detection
at the initial trajectory (a0), K ADMM iterations (a1-a8: pair sweep with fused
multiplier update, Riccati primal step), final multiplier update, and scale
detection at the final trajectory.

Workload (default): BASELINE.json configs[4] = C5, 4096 independent scenes x 200
obstacles x N = 50, K = 100 per GPU (weak scaling: rank r solves scenes
[4096 r, 4096 (r+1)); scenes are independent, so there is no data-path
collective -- torch.distributed is used for the barrier and the max-over-ranks
timer only).  Inputs (5.6 GB of resident iterate) exceed the 126 MB L2.

    python bench.py [--gpus N --steps K --warmup W] [--impl reference]
    python -m torch.distributed.run --nproc-per-node N ... bench.py --gpus N
    python bench.py --config 4 --shard obstacles   # one problem split across GPUs by
                                                   # obstacle blocks (ncclAllReduce/iter)

Prints ONE JSON line (rank 0).
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
# stdout carries exactly one JSON line: main() moves file descriptor 1 onto stderr
# (NCCL's version banner, library chatter) and keeps a private handle for emit()
_JSON_OUT = None


def emit(line: dict):
    out = _JSON_OUT or sys.stdout
    out.write(json.dumps(line) + "\n")
    out.flush()

import scenes  # noqa: E402  (seeded generators: shared by both arms)

MEASURED = os.path.join(ROOT, "MEASURED_PEAKS.json")
PROFILE_SUMMARY = os.path.join(ROOT, "profiles", "traffic.json")


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", type=int, default=5)
    ap.add_argument("--shard", default="scenes", choices=["scenes", "obstacles"],
                    help="multi-GPU split: independent scenes per rank (no collective, weak scaling) or the "
                         "obstacles of one problem (one ncclAllReduce per iteration, strong scaling)")
    ap.add_argument("--scenes", type=int, default=scenes.C5_SCENES, help="C5 scenes per rank")
    ap.add_argument("--iters", type=int, default=0, help="ADMM iterations per solve (0 = config default)")
    ap.add_argument("--e2e-steps", type=int, default=2)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--prox-eps", type=float, default=0.0,
                    help="reading #2 proximal term (0 = paper-exact Eq. 19); > 0 runs the NEXT f4 dual Newton")
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def make_scene(cfg, rank, n_scenes):
    if cfg == 5:
        return scenes.make_c5(scene_ids=range(rank * n_scenes, (rank + 1) * n_scenes))
    return scenes.make_config(cfg)


def slice_obstacles(sc, j0, j1):
    """The same problem restricted to obstacles [j0, j1) of every scene (rank-local view)."""
    import dataclasses

    M = sc.n_obs
    offs, Cs, ds = [0], [], []
    for b in range(sc.n_scenes):
        for j in range(j0, j1):
            lo, hi = sc.obs_off[b * M + j], sc.obs_off[b * M + j + 1]
            Cs.append(sc.obs_C[lo:hi])
            ds.append(sc.obs_d[lo:hi])
            offs.append(offs[-1] + hi - lo)
    step = None
    if sc.obs_step is not None:
        step = np.concatenate([sc.obs_step[b * M + j0:b * M + j1] for b in range(sc.n_scenes)])
    return dataclasses.replace(sc, n_obs=j1 - j0, obs_off=np.asarray(offs, np.int32),
                               obs_C=np.concatenate(Cs) if Cs else np.zeros((0, sc.dim)),
                               obs_d=np.concatenate(ds) if ds else np.zeros(0), obs_step=step)


def workload_name(cfg, n_scenes, iters, prox_eps=0.0):
    # prox_eps > 0: the proximal variant of reading #2 (NEXT f4 dual Newton), not the paper's Eq. 19
    px = f", prox_eps={prox_eps:g} (NEXT f4)" if prox_eps > 0 else ""
    if cfg == 5:
        return f"C5: {n_scenes} scenes x 200 obstacles x N=50 per GPU, K={iters} ADMM iterations" + px
    return scenes.CONFIG_NAMES[cfg].split(",")[0] + f", K={iters}" + px


# ----------------------------------------------------------------------------
# measurement helpers
# ----------------------------------------------------------------------------

class Clocks:
    """nvidia-smi sampling DURING the timed region (B200_PROFILING.md clocks line)."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, dev):
        self.dev = dev
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.dev), f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"]}
        self.proc.terminate()
        out, _ = self.proc.communicate(timeout=10)
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in out.strip().splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) < 8:
                continue
            try:
                sm.append(float(f[0]))
                smax.append(float(f[1]))
            except ValueError:
                continue
            for nm, v in zip(names, f[4:8]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        load = [x for x in sm if x > 500] or sm
        return {"sm_mhz": float(np.median(load)) if load else None,
                "sm_max_mhz": max(smax) if smax else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def hbm_peak():
    try:
        return float(json.load(open(MEASURED))["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


def algorithmic_bytes_per_sweep(sc):
    """HBM bytes one pair-sweep launch must move: per pair read
    y^k (n_p doubles), zeta, xi (1+d) and write y^{k+1}, zeta, xi (fused multiplier
    update) + a 4-byte pivot/status word; per scene the obstacle faces once
    ((d+1) doubles per face); per (scene, t, chunk) one 20-double record."""
    n = sc.lcp_sizes().astype(np.float64)
    d = sc.dim
    per_pair = 16.0 * n.sum() + sc.n_pairs * (16.0 * (1 + d) + 4.0)
    faces = float(sc.obs_off[-1]) * 8.0 * (d + 1)
    G = sc.n_parts * sc.n_obs
    nchunk = max(1, -(-G // 32))  # one-warp CTAs
    recs = sc.n_scenes * sc.horizon * nchunk * 20 * 8.0
    return per_pair + faces + recs


def algorithmic_flops_per_sweep(sc, pivots_per_sweep):
    """FP64 flops of the revised Lemke sweep, FMA = 2:
    setup per pair 2[n_o(d + d^2) + (n_r-1) d + (n-1)(d+1)]; per pivot 2(d+2)n + 2n
    (entering column of every basic variable + right-hand-side update)."""
    d = sc.dim
    n = sc.lcp_sizes().astype(np.float64)
    nr = np.diff(sc.part_off)
    no = np.diff(sc.obs_off).reshape(sc.n_scenes, sc.n_obs)
    no_p = np.broadcast_to(no[:, None, None, :], (sc.n_scenes, sc.horizon, sc.n_parts, sc.n_obs)).reshape(-1)
    nr_p = np.broadcast_to(nr[None, None, :, None], (sc.n_scenes, sc.horizon, sc.n_parts, sc.n_obs)).reshape(-1)
    setup = 2.0 * (no_p * (d + d * d) + (nr_p - 1) * d + (n - 1) * (d + 1)).sum()
    nbar = n.mean()
    per_pivot = 2.0 * (d + 2) * nbar + 2.0 * nbar
    return setup + pivots_per_sweep * per_pivot


def pinned_scene(sc):
    """Copy the per-batch input arrays into pinned host memory (torch) for the e2e leg."""
    import dataclasses

    import torch

    def pin(a):
        t = torch.from_numpy(np.ascontiguousarray(a)).pin_memory()
        return t.numpy()

    fields = ("part_off", "part_A", "part_b", "obs_off", "obs_C", "obs_d", "dyn_A", "dyn_B", "dyn_c", "Qs",
              "Qu", "s0", "s_ref")
    return dataclasses.replace(sc, **{f: pin(getattr(sc, f)) for f in fields})


def h2d_bytes(sc):
    rows_o = int(sc.obs_off[-1])
    rows_p = int(sc.part_off[-1])
    b = 32 * rows_o + 32 * rows_p + 4 * (len(sc.obs_off) + len(sc.part_off))
    b += 8 * (sc.dyn_A.size + sc.dyn_B.size + sc.dyn_c.size + sc.Qs.size + sc.Qu.size + sc.s0.size)
    b += 8 * 2 * sc.s_ref.size  # s_ref and the initial trajectory
    return int(b)


# ----------------------------------------------------------------------------
# the reference arm: the CPU oracle (test infrastructure), bounded sample
# ----------------------------------------------------------------------------

def oracle_sample(cfg, iters, prox_eps=0.0):
    """Time the oracle as it stands on one scene of the workload (single thread)."""
    import oracle

    sc = make_scene(cfg, 0, 1) if cfg == 5 else make_scene(cfg, 0, 1)
    o = oracle.Oracle(sc, prox_eps=prox_eps)
    t0 = time.perf_counter()
    o.scale_detect()
    o.admm_iterate(iters)
    o.scale_detect()
    dt = time.perf_counter() - t0
    return sc.n_pairs * iters / dt, dt, sc


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


def run_reference(args, rank, world):
    if rank != 0:
        return
    cfg = args.config
    iters_full = args.iters or (100 if cfg == 5 else scenes.make_config(cfg).iters)
    sample_iters = min(iters_full, 20)
    for _ in range(args.warmup):
        oracle_sample(cfg, max(1, sample_iters // 4), args.prox_eps)
    vals, ts = [], []
    sc = None
    for _ in range(args.steps):
        v, dt, sc = oracle_sample(cfg, sample_iters, args.prox_eps)
        vals.append(v)
        ts.append(dt)
    value = float(np.median(vals))
    sample = (f"1 scene ({sc.n_pairs // max(1, sc.horizon)} pairs/timestep x N={sc.horizon}, "
              f"{sc.n_pairs} pair-QPs/iter) x {sample_iters} ADMM iterations + 2 scale detections per step; "
              f"oracle/liborc.so single-threaded on {cpu_model()}")
    line = {
        "impl": "reference", "metric": "pair-QPs/sec", "value": value, "unit": "pair-QP/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": float(np.mean(ts) * 1e3), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded scenes/ generators)",
        "config": {"workload": workload_name(cfg, args.scenes if cfg == 5 else 1, iters_full, args.prox_eps),
                   "sample": "bounded CPU sample (see cpu_baseline.sample)"},
        "cpu_baseline": {"value": value, "unit": "pair-QP/s", "cores": 1, "kind": "oracle", "sample": sample},
        "e2e": {"value": value, "unit": "pair-QP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    emit(line)


# ----------------------------------------------------------------------------
# our arm
# ----------------------------------------------------------------------------

def run_ours(args, rank, world, local):
    import torch

    import paper_2406_07048_b200 as ca

    if not torch.cuda.is_available():
        raise SystemExit("bench.py: no CUDA device -- this implementation has no CPU fallback")
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    stream = torch.cuda.current_stream()
    cfg = args.config
    obstacle_shard = args.shard == "obstacles"
    if obstacle_shard:
        # every rank holds the same problem and solves its obstacle block
        sc = make_scene(cfg, 0, args.scenes)
        nid = ca.nccl_unique_id() if rank == 0 else None
        if dist:
            box = [nid]
            dist.broadcast_object_list(box, src=0)
            nid = box[0]
        g = ca.Problem(sc, device=local, stream=stream.cuda_stream, dist=(world, rank, nid), workspace="torch",
                       prox_eps=args.prox_eps)
        sc_local = slice_obstacles(sc, g.j0, g.j1)
    else:
        sc = make_scene(cfg, rank, args.scenes)
        g = ca.Problem(sc, device=local, stream=stream.cuda_stream, workspace="torch", prox_eps=args.prox_eps)
        sc_local = sc
    iters = args.iters or sc.iters
    fp64 = ca.fp64_peak(local, 300.0) if rank == 0 else None

    def step():
        g.reset_iterate()
        g.scale_detect(want_alpha=False)
        g.admm_iterate(iters, hist=False)
        _, amin = g.scale_detect(want_alpha=False)
        return amin

    def barrier():
        if dist:
            dist.barrier()
        torch.cuda.synchronize()

    for _ in range(args.warmup):
        step()
    g.set_timing(True)
    g.kernel_times(reset=True)
    clocks = Clocks(local)
    barrier()
    clocks.start()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        amin = step()
    e1.record(stream)
    torch.cuda.synchronize()
    clk = clocks.stop()
    barrier()
    ms = e0.elapsed_time(e1)
    kt = g.kernel_times(reset=True)
    g.set_timing(False)
    if dist:
        t = torch.tensor([ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    units = 1 if obstacle_shard else world  # obstacle sharding splits ONE problem
    pairs_total = sc.n_pairs * iters * args.steps * units
    value = pairs_total / (ms * 1e-3)
    solves = sc.n_scenes * args.steps * units / (ms * 1e-3)
    launches = int(sum(v[1] for v in kt.values()))
    # pivots of the last solve (for the algorithmic flop count; rank-local pairs)
    g.reset_iterate()
    rc, hist = g.admm_iterate(iters, hist=True)
    piv_per_sweep = float(hist["pivots"].mean())
    fails = int(hist["n_fail"].sum())

    # e2e through the public API with host buffers: load (H2D) + solve + D2H
    e2e = None
    if not args.no_e2e:
        psc = pinned_scene(sc)
        s_host = torch.empty((sc.n_scenes, sc.horizon + 1, sc.n_state), dtype=torch.float64).pin_memory().numpy()

        def e2e_step():
            g.load(psc)
            g.scale_detect(want_alpha=False)
            g.admm_iterate(iters, hist=False)
            s, u = g.trajectory()
            _, amin = g.scale_detect(want_alpha=False)
            return s, u, amin

        e2e_step()
        barrier()
        t0 = time.perf_counter()
        for _ in range(args.e2e_steps):
            e2e_step()
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        if dist:
            t = torch.tensor([dt], device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            dt = float(t.item())
        e2e = {"value": sc.n_pairs * iters * args.e2e_steps * units / dt, "unit": "pair-QP/s",
               "h2d_bytes_per_step": h2d_bytes(sc),
               "d2h_bytes_per_step": int(8 * (sc.n_scenes * (sc.horizon + 1) * sc.n_state
                                              + sc.n_scenes * sc.horizon * sc.n_ctrl + 2 * sc.n_scenes)),
               "steps": args.e2e_steps,
               "what": "ca_problem_load from pinned host arrays + 2 scale detects + K iterations + "
                       "ca_get_trajectory (host), wall clock, max over ranks"}

    if rank != 0:
        return
    sweep_ms, sweep_n = kt["sweep"]
    avg_sweep_ms = sweep_ms / max(1, sweep_n)
    nbytes = algorithmic_bytes_per_sweep(sc_local)
    flops = algorithmic_flops_per_sweep(sc_local, piv_per_sweep)
    hbm, hbm_src = hbm_peak()
    achieved_gbs = nbytes / (avg_sweep_ms * 1e-3) / 1e9
    achieved_tf = flops / (avg_sweep_ms * 1e-3) / 1e12
    traffic = None
    try:
        prof = json.load(open(PROFILE_SUMMARY))
        if prof.get("workload_key") == f"C{cfg}-{sc.n_scenes}" and not obstacle_shard:
            traffic = prof.get("sweep_dram_bytes_per_launch")
    except Exception:
        pass
    frac_hbm = achieved_gbs / hbm
    frac_fp = achieved_tf / fp64 if fp64 else 0.0
    if frac_hbm >= frac_fp:
        roof = {"bound": "hbm", "achieved": achieved_gbs, "peak": hbm, "unit": "GB/s", "frac": frac_hbm,
                "traffic": traffic, "peak_source": hbm_src}
    else:
        roof = {"bound": "alu", "achieved": achieved_tf, "peak": fp64, "unit": "TFLOP/s", "frac": frac_fp,
                "traffic": traffic, "peak_source": "measured FP64 DFMA loop (ca_fp64_peak)"}
    roof.update({"kernel": "k_sweep (ADMM step 1 + fused step 3)", "launch_ms": avg_sweep_ms,
                 "pair_solver": ("dual semismooth Newton (NEXT f4; 'pivots' = Newton iterations, the flop "
                                 "model is the revised Lemke's, indicative only)") if args.prox_eps > 0
                                else "revised Lemke (paper-exact Eq. 19)",
                 "algorithmic_bytes_per_launch": nbytes, "algorithmic_flops_per_launch": flops,
                 "hbm_frac": frac_hbm, "fp64_frac": frac_fp, "fp64_peak_tflops": fp64,
                 "pivots_per_pair": piv_per_sweep / max(1, sc_local.n_pairs),
                 "share_of_step": sweep_ms / ms if ms else None})
    cpu = None
    if world == 1 and not args.no_cpu:
        v, dt, ssc = oracle_sample(cfg, min(iters, 100), args.prox_eps)
        cpu = {"value": v, "unit": "pair-QP/s", "cores": 1, "kind": "oracle",
               "sample": f"scene 0 alone ({ssc.n_pairs} pair-QPs/iter) x {min(iters, 100)} ADMM iterations "
                         f"+ 2 scale detections, {dt:.1f} s single-threaded on {cpu_model()}"}
    line = {
        "metric": "pair-QPs/sec", "value": value, "unit": "pair-QP/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
        "scaling": "strong" if obstacle_shard else "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded scenes/ generators)",
        "config": {"workload": workload_name(cfg, sc.n_scenes, iters, args.prox_eps), "scenes_per_gpu": sc.n_scenes,
                   "admm_iters": iters, "pair_qps_per_iter_per_gpu": sc.n_pairs,
                   "parallelism": (f"obstacle-sharded x{world}, one ncclAllReduce of per-(scene,t) aggregates "
                                   f"per iteration" if obstacle_shard else
                                   f"scene-sharded x{world}, no data-path collective"),
                   "l2": "inputs larger than L2 (resident iterate %.1f GB)" % (g.device_bytes / 1e9)},
        "admm_solves_per_sec": solves,
        "kernel_ms_per_step": {k: v[0] / args.steps for k, v in kt.items()},
        "roofline": roof, "cpu_baseline": cpu, "e2e": e2e, "clocks": clk, "gpu_launches": launches,
        "lemke_failures": fails, "min_alpha_final": float(np.min(amin)),
    }
    emit(line)


def main():
    global _JSON_OUT
    _JSON_OUT = os.fdopen(os.dup(1), "w")
    sys.stdout.flush()
    os.dup2(2, 1)
    args = parse()
    rank, world, local = dist_env()
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    run_ours(args, rank, world, local)


if __name__ == "__main__":
    main()
