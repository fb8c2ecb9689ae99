#!/usr/bin/env python
"""Benchmark of the ADMM hot path of arXiv 2406.07048 on B200 (sm_100a, FP64).

One *step* = one full ADMM solve of the whole hot path over one batch (SURVEY
§8(a)): reset to the initial iterate (O1), scale detection
at the initial trajectory (a0), K ADMM iterations (a1-a8: pair sweep with fused
multiplier update, Riccati primal step), final multiplier update, and scale
detection at the final trajectory.

Workload (default): BASELINE.json configs[4] = C5, 4096 independent scenes x 200
obstacles x N = 50, K = 100.  On N GPUs the SAME 4096 scenes are split over the ranks
(strong scaling, the scene grid of include/ca.h ca_dist_desc: rank r solves scenes
[4096 r / N, 4096 (r+1) / N)) with ONE ncclAllReduce per ADMM iteration of every
scene's Eq. 18 statistics (global residuals on every rank, BASELINE config 5).
--shard weak: 4096 scenes PER rank, no data-path collective (weak scaling);
--shard obstacles: one problem split by obstacle blocks (ncclAllReduce of the
per-(scene, t) aggregates per iteration).  Inputs (>= 5 GB of resident iterate at
N = 1) exceed the 126 MB L2.

    python bench.py [--gpus N --steps K --warmup W] [--impl reference]
    python bench.py --gpus 8        # spawns 8 ranks itself (torch.distributed.run)
    python -m torch.distributed.run --nproc-per-node N ... bench.py --gpus N
    python bench.py --config 4 --shard obstacles
    python bench.py --config 2      # C1-C4: one scene, full K, oracle at full K

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
    ap.add_argument("--shard", default="scenes", choices=["scenes", "weak", "obstacles"],
                    help="multi-GPU split: the batch's scenes over the ranks with a per-iteration allreduce of "
                         "per-scene statistics (strong scaling, default), independent scene batches per rank "
                         "(weak scaling, no collective), or the obstacles of one problem (strong scaling, one "
                         "ncclAllReduce of the aggregates per iteration)")
    ap.add_argument("--scenes", type=int, default=scenes.C5_SCENES,
                    help="C5 scenes: of the whole job (scenes / obstacles sharding), per rank (weak)")
    ap.add_argument("--iters", type=int, default=0, help="ADMM iterations per solve (0 = config default)")
    ap.add_argument("--e2e-steps", type=int, default=2)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--prox-eps", type=float, default=0.0,
                    help="reading #2 proximal term (0 = paper-exact Eq. 19); > 0 runs the NEXT f4 dual Newton")
    ap.add_argument("--force-dist", action="store_true",
                    help="at one GPU, run the --shard mode's multi-GPU code path anyway (NCCL communicator of one "
                         "rank; scenes mode sets CA_FORCE_SCENE_GRID=1 so the per-iteration scene exchange runs)")
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def make_scene(cfg, rank, n_scenes):
    """C5: scenes [rank n, (rank+1) n) (a weak-scaling rank's own batch; rank 0 = the
    first n scenes); other configs: the single-scene problem."""
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


def workload_name(cfg, n_scenes, iters, prox_eps=0.0, per_gpu=False):
    # prox_eps > 0: the proximal variant of reading #2 (NEXT f4 dual Newton), not the paper's Eq. 19
    px = f", prox_eps={prox_eps:g} (NEXT f4)" if prox_eps > 0 else ""
    if cfg == 5:
        return (f"C5: {n_scenes} scenes x 200 obstacles x N=50{' per GPU' if per_gpu else ''}, "
                f"K={iters} ADMM iterations" + px)
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
    """HBM bytes one pair-sweep launch must move: per pair read y^k (n_p
    doubles), zeta, xi (1+d) and write y^{k+1}, zeta, xi (fused multiplier update) + a
    4-byte pivot/status word; per scene the obstacle faces once ((d+1) doubles per face);
    one record of (d+1)(d+2)/2 + (d+1) + 8 doubles per (work item, timestep slot) -- the
    library's layout: sort pools of TG timesteps (TG = min(8, 800 // (parts x obstacles))
    when the sweep spans >= 10000 items of 32 pairs, else 1), chunks of 32 pairs."""
    n = sc.lcp_sizes().astype(np.float64)
    d = sc.dim
    per_pair = 16.0 * n.sum() + sc.n_pairs * (16.0 * (1 + d) + 4.0)
    faces = float(sc.obs_off[-1]) * 8.0 * (d + 1)
    G = sc.n_parts * sc.n_obs
    nchunk = max(1, -(-G // 32))
    items1 = sc.n_scenes * sc.horizon * nchunk
    TG = min(8, max(1, min(sc.horizon, 800 // max(1, G)))) if items1 >= 10000 else 1
    NG = -(-sc.horizon // TG)
    nchunkG = -(-(TG * max(1, G)) // 32)
    rec = (d + 1) * (d + 2) // 2 + (d + 1) + 8
    recs = sc.n_scenes * NG * nchunkG * TG * rec * 8.0
    return per_pair + faces + recs


def algorithmic_flops_per_sweep(sc, pivots_per_sweep):
    """FP64 flops of one pair sweep by SURVEY §8(d)'s model (the contract's algorithmic
    count, FMA = 2, division = 1), per pair with n = n_r + n_o + 1 and p its pivots:
      F0   = 2 [(n-1) n / 2 (d+1) + 2 (n-1)(d+1) + n_o d (d+1)] + 70 + 50
             (M = Kt Kt^T and q, elimination, obstacle rows at the pose; multiplier update;
              recovery and aggregates)
      Fpiv = 2 n (n + 2) + n        (one pivot of the compact tableau)
    summed over pairs with the measured mean pivots per pair."""
    d = sc.dim
    n = sc.lcp_sizes().astype(np.float64)
    no = np.diff(sc.obs_off).reshape(sc.n_scenes, sc.n_obs)
    no_p = np.broadcast_to(no[:, None, None, :], (sc.n_scenes, sc.horizon, sc.n_parts, sc.n_obs)).reshape(-1)
    f0 = (2.0 * ((n - 1) * n / 2 * (d + 1) + 2 * (n - 1) * (d + 1) + no_p * d * (d + 1)) + 120.0).sum()
    p = pivots_per_sweep / max(1, sc.n_pairs)
    fpiv = (2.0 * n * (n + 2) + n).sum() * p
    return f0 + fpiv


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

def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


def host_cores():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def oracle_rates(cfg, iters, prox_eps=0.0, budget_s=20.0):
    """The CPU oracle as it stands (test infrastructure, oracle/liborc.so), timed on this
    box's host cores on a bounded sample of the workload:
      one core:  C5 -- one scene, C1-C4 -- the whole problem; at up to `iters` iterations
      all cores: C5 -- one scene per core fanned out over scenes (POSIX threads,
                 orc_admm_iterate_mt: bitwise the sequential run), C1-C4 -- the pairs of
                 each dual step fanned out over the cores.
    Both include the two scale detections of a step.  Returns a cpu_baseline dict."""
    import oracle

    ncores = host_cores()

    def timed(sc, k, threads):
        o = oracle.Oracle(sc, prox_eps=prox_eps)
        t0 = time.perf_counter()
        o.scale_detect()
        if threads > 1:
            o.admm_iterate_mt(k, threads)
        else:
            o.admm_iterate(k)
        o.scale_detect()
        return time.perf_counter() - t0

    if cfg == 5:
        one = make_scene(5, 0, 1)
        k1 = min(iters, 20)
        t1 = timed(one, k1, 1)
        v1 = one.n_pairs * k1 / t1
        many = make_scene(5, 0, ncores)
        # enough iterations for ~budget/2 seconds of all-core work (the rate per core is v1)
        km = int(max(2, min(iters, 0.5 * budget_s * v1 / many.n_pairs * ncores)))
        tm = timed(many, km, ncores)
        vm = many.n_pairs * km / tm
        s1 = f"scene 0 alone ({one.n_pairs} pair-QPs/iter) x {k1} ADMM iterations + 2 scale detections, {t1:.2f} s"
        sm = (f"scenes 0..{ncores - 1} ({many.n_pairs} pair-QPs/iter) x {km} iterations + 2 scale detections, "
              f"{ncores} threads over scenes, {tm:.2f} s")
    else:
        sc = make_scene(cfg, 0, 1)
        t1 = timed(sc, iters, 1)
        v1 = sc.n_pairs * iters / t1
        # threads over the pairs of each dual step: one per ~500 pairs (a thread start per
        # iteration costs more than a few hundred tiny pair QPs)
        ncores = max(1, min(ncores, sc.n_pairs // 500))
        tm = timed(sc, iters, ncores) if ncores > 1 else t1
        vm = sc.n_pairs * iters / tm
        s1 = f"the whole problem ({sc.n_pairs} pair-QPs/iter) x K={iters} (full K) + 2 scale detections, {t1:.2f} s"
        sm = f"the same, {ncores} thread(s) over the pairs of each dual step, {tm:.2f} s"
    return {"value": vm, "unit": "pair-QP/s", "cores": ncores, "kind": "oracle",
            "sample": f"all cores: {sm}; one core: {s1}; {cpu_model()}, {host_cores()} host cores",
            "single_core": {"value": v1, "unit": "pair-QP/s", "cores": 1, "sample": s1},
            "cpu_model": cpu_model(), "hardware_concurrency": os.cpu_count()}


def run_reference(args, rank, world):
    """--impl reference: the oracle as it stands, all host cores, each step a bounded
    sample of this config's workload (the reference arm of this tier); rank 0 only."""
    if rank != 0:
        return
    cfg = args.config
    iters_full = args.iters or (100 if cfg == 5 else scenes.make_config(cfg).iters)
    for _ in range(args.warmup):
        oracle_rates(cfg, max(1, min(iters_full, 20) // 4), args.prox_eps, budget_s=2.0)
    vals, ts, cb = [], [], None
    for _ in range(args.steps):
        t0 = time.perf_counter()
        cb = oracle_rates(cfg, iters_full if cfg != 5 else 100, args.prox_eps, budget_s=6.0)
        ts.append(time.perf_counter() - t0)
        vals.append(cb["value"])
    value = float(np.median(vals))
    cb = dict(cb, value=value)
    line = {
        "impl": "reference", "metric": "pair-QPs/sec", "value": value, "unit": "pair-QP/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": float(np.mean(ts) * 1e3), "higher_is_better": True,
        "scaling": "strong" if cfg != 5 or args.shard != "weak" else "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded scenes/ generators)",
        "config": {"workload": workload_name(cfg, args.scenes if cfg == 5 else 1, iters_full, args.prox_eps),
                   "sample": "bounded CPU sample (see cpu_baseline.sample)"},
        "cpu_baseline": cb,
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
    mode = args.shard if world > 1 or args.force_dist else "single"
    if cfg != 5 and mode == "scenes":
        mode = "obstacles"  # one scene: its obstacles are what can be split
    if mode in ("scenes", "obstacles"):
        # every rank holds the FULL problem; the library keeps this rank's block of the
        # scene x obstacle grid (include/ca.h ca_dist_desc) and exchanges one allreduce
        # per ADMM iteration over NCCL
        sc = make_scene(cfg, 0, args.scenes)
        nid = ca.nccl_unique_id() if rank == 0 else None
        if world > 1:
            box = [nid]
            dist.broadcast_object_list(box, src=0)
            nid = box[0]
        elif mode == "scenes":
            os.environ["CA_FORCE_SCENE_GRID"] = "1"
        grid = (world, 1) if mode == "scenes" else (1, world)
        g = ca.Problem(sc, device=local, stream=stream.cuda_stream, dist=(world, rank, nid, *grid),
                       workspace="torch", prox_eps=args.prox_eps)
        sc_local = slice_obstacles(g.sc, g.j0, g.j1) if mode == "obstacles" else g.sc
    else:  # one GPU, or weak scaling: this rank's own independent batch
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
    units = world if mode == "weak" else 1  # weak: every rank its own batch; else ONE batch split
    pairs_total = sc.n_pairs * iters * args.steps * units
    value = pairs_total / (ms * 1e-3)
    solves = sc.n_scenes * args.steps * units / (ms * 1e-3)
    launches = int(sum(v[1] for k, v in kt.items() if k != "comm"))  # this library's kernels (NCCL apart)
    # pivots of the last solve (for the algorithmic flop count; rank-local pairs)
    g.reset_iterate()
    rc, hist = g.admm_iterate(iters, hist=True)
    piv_per_sweep = float(hist["pivots"].mean())
    if mode == "scenes":  # the history is global there: this rank's share of the pivots
        piv_per_sweep *= sc_local.n_pairs / sc.n_pairs
    fails = int(hist["n_fail"].sum())
    fail_kinds = {k: int(hist[k].sum()) for k in ("n_ray", "n_iterlimit", "n_neg_ye")}
    max_piv = int(hist["max_pivots"].max())

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
               "h2d_bytes_per_step": h2d_bytes(sc) * units,
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
        if prof.get("workload_key") == f"C{cfg}-{sc_local.n_scenes}" and mode != "obstacles":
            traffic = prof.get("sweep_dram_bytes_per_launch")
    except Exception:
        pass
    frac_hbm = achieved_gbs / hbm
    frac_fp = achieved_tf / fp64 if fp64 else 0.0
    if frac_hbm >= frac_fp:
        roof = {"bound": "hbm", "achieved": achieved_gbs, "peak": hbm, "unit": "GB/s", "frac": frac_hbm,
                "traffic": traffic, "peak_source": hbm_src}
    else:  # the FP64 vector pipe (no tensor cores: not a dense contraction)
        roof = {"bound": "alu", "achieved": achieved_tf, "peak": fp64, "unit": "TFLOP/s", "frac": frac_fp,
                "traffic": traffic,
                "peak_source": "measured FP64 DFMA loop on all SMs (ca_fp64_peak); unit count: 148 SMs x 64 DFMA/clk "
                               "x 2 x 1.965 GHz = 37.2 TFLOP/s"}
    roof.update({"kernel": "k_sweep (ADMM step 1 + fused step 3)", "launch_ms": avg_sweep_ms,
                 "flop_model": "SURVEY 8(d): 2[(n-1)n/2 (d+1) + 2(n-1)(d+1) + n_o d(d+1)] + 120 per pair + "
                               "(2n(n+2) + n) per pivot, measured pivots",
                 "pair_solver": ("dual semismooth Newton (NEXT f4; 'pivots' = Newton iterations, the flop "
                                 "model is Lemke's, indicative only)") if args.prox_eps > 0
                                else "revised Lemke (paper-exact Eq. 19)",
                 "algorithmic_bytes_per_launch": nbytes, "algorithmic_flops_per_launch": flops,
                 "hbm_frac": frac_hbm, "fp64_frac": frac_fp, "fp64_peak_tflops": fp64,
                 "pivots_per_pair": piv_per_sweep / max(1, sc_local.n_pairs),
                 "share_of_step": sweep_ms / ms if ms else None})
    cpu = None
    if world == 1 and not args.no_cpu:
        cpu = oracle_rates(cfg, iters, args.prox_eps)
    par = {"single": "one GPU",
           "scenes": f"scene-sharded x{world} (one batch split by scenes), one ncclAllReduce of every scene's "
                     f"Eq. 18 statistics per iteration",
           "weak": f"weak x{world} (every rank its own {sc.n_scenes}-scene batch), no data-path collective",
           "obstacles": f"obstacle-sharded x{world}, one ncclAllReduce of per-(scene,t) aggregates per iteration"}[mode]
    line = {
        "metric": "pair-QPs/sec", "value": value, "unit": "pair-QP/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
        "scaling": "weak" if mode == "weak" else "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded scenes/ generators)",
        "config": {"workload": workload_name(cfg, sc.n_scenes, iters, args.prox_eps, per_gpu=mode == "weak"),
                   "scenes_total": sc.n_scenes * units, "scenes_per_gpu": sc_local.n_scenes,
                   "admm_iters": iters, "pair_qps_per_iter_per_gpu": sc_local.n_pairs, "parallelism": par,
                   "l2": "inputs larger than L2 (resident iterate %.1f GB per GPU)" % (g.device_bytes / 1e9),
                   **({"force_dist": True} if args.force_dist and world == 1 else {})},
        "admm_solves_per_sec": solves,
        "kernel_ms_per_step": {k: v[0] / args.steps for k, v in kt.items()},
        "roofline": roof, "cpu_baseline": cpu, "e2e": e2e, "clocks": clk, "gpu_launches": launches,
        "nccl_collectives": int(kt["comm"][1]),
        "lemke_failures": fails, "lemke_failure_kinds": fail_kinds, "max_pivots": max_piv,
        "min_alpha_final": float(np.min(amin)),
    }
    emit(line)


def spawn_ranks(args):
    """--gpus N > 1 without a torchrun environment: launch the N ranks ourselves (one
    process per GPU, torch.distributed.run, rendezvous on 127.0.0.1); rank 0's JSON line
    comes through our stdout."""
    import socket

    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__), *sys.argv[1:]]
    return subprocess.call(cmd)


def main():
    global _JSON_OUT
    args = parse()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(spawn_ranks(args))
    _JSON_OUT = os.fdopen(os.dup(1), "w")
    sys.stdout.flush()
    os.dup2(2, 1)
    rank, world, local = dist_env()
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE {world}")
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    run_ours(args, rank, world, local)


if __name__ == "__main__":
    main()
