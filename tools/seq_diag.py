"""cfg1-budget sequence on the GPU vs the reference golden: data-term traces at checkpoints (debug)."""
import sys
sys.path.insert(0, ".")
import numpy as np
from paper_2507_14046_b200 import reconstruct_sequence, RunConfig
from paper_2507_14046_b200 import workloads as W
g = np.load("tests/golden/seq_cfg1.npz")
spec = W.CONFIGS["cfg1"]
wl = W.make_workload(spec, seed=0, frames=4)
for prec in sys.argv[1:] or ["tf32"]:
    cfg = W.run_config_for(spec, tuple(g["output_map"]), seed=0, precision=prec)
    res = reconstruct_sequence(wl.matrix, wl.voltages, cfg, wl.grid)
    w = res.traces["warm"].data_terms()
    ck = [0, 9, 49, 99, 199, 499, 999, 1499, 1999]
    print(prec, "warm  gpu", " ".join(f"{w[k]:.4g}" for k in ck))
    print(prec, "warm  ref", " ".join(f"{g['trace_warm'][k]:.4g}" for k in ck))
    print(prec, "warm band", " ".join(f"{g['band_trace_warm'][k]:.4g}" for k in ck))
    for i in range(1, 5):
        t = res.traces[f"frame_{i}"].data_terms()
        print(prec, f"frame {i} gpu {t[0]:.4g} -> {t[-1]:.4g}  ref {g[f'trace_frame_{i}'][0]:.4g} -> {g[f'trace_frame_{i}'][-1]:.4g}"
              f"  band {g[f'band_trace_frame_{i}'][0]:.4g} -> {g[f'band_trace_frame_{i}'][-1]:.4g}")
