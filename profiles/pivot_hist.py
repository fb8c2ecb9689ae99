"""Lemke pivot-count histograms (they feed the algorithmic flop model).
GPU: C5 (4096 scenes, K = 100) -- histogram of every pair's pivots at sweeps 1, 10, 50,
100 and the mean per sweep; oracle: C1-C4 at full K, histogram of the last sweep and the
mean over all sweeps.  Writes profiles/r02/pivot_hist.json."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

import scenes  # noqa: E402

out = {}
if "--gpu" in sys.argv:
    import paper_2406_07048_b200 as ca

    sc = scenes.make_c5()
    g = ca.Problem(sc)
    K = 100
    hists, means = {}, []
    for k in range(1, K + 1):
        rc, h = g.admm_iterate(1)
        means.append(float(h["pivots"][0]) / sc.n_pairs)
        if k in (1, 10, 50, 100):
            piv = np.concatenate([g.pair_state(p0, min(4_000_000, g.n_pairs - p0), fields=("pivots",))["pivots"]
                                  for p0 in range(0, g.n_pairs, 4_000_000)])
            hists[k] = np.bincount(piv).tolist()
    out["C5_gpu"] = {"pairs": sc.n_pairs, "hist_at_sweep": hists, "mean_per_sweep": means,
                     "mean_all": float(np.mean(means))}
else:
    import oracle

    for cfg in (1, 2, 3, 4):
        sc = scenes.make_config(cfg)
        o = oracle.Oracle(sc)
        tot = []
        for k in range(sc.iters):
            o.dual_sweep()
            tot.append(float(o.pivots[: sc.n_pairs].mean()))
            o.primal_step()
            o.multiplier_update()
        out[f"C{cfg}_oracle"] = {"pairs": sc.n_pairs, "K": sc.iters,
                                 "hist_last_sweep": np.bincount(o.pivots[: sc.n_pairs]).tolist(),
                                 "mean_all": float(np.mean(tot)), "lcp_n": sorted(set(sc.lcp_sizes().tolist()))}
dst = os.path.join(ROOT, "gpurun_out" if "--gpu" in sys.argv else "profiles", "r02")  # GPU runs: brought back
os.makedirs(dst, exist_ok=True)
name = "pivot_hist_gpu_c5.json" if "--gpu" in sys.argv else "pivot_hist_oracle_c1_c4.json"
json.dump(out, open(os.path.join(dst, name), "w"), indent=1)
print({k: v.get("mean_all") for k, v in out.items()})
