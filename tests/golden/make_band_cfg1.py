"""More members of the cfg1-budget variability band (tests/golden/seq_cfg1_band.npz).

seq_cfg1.npz holds the real reference's run (dense operator, all host threads) and ONE
reordering of the same arithmetic (the oracle -- bit-exact with the reference on the golden
cases -- with the compact operator). This script adds reorderings that change nothing but the
host thread count (the CPU convolution / reduction partitioning, hence the fp32 summation
order): the oracle with the compact operator at 2, 4 and 8 threads (8 reproduces the band of
seq_cfg1.npz bit for bit on an 8-core host). The GPU test judges its
distance from the reference against the spread of ALL these reference-side reorderings.

Needs only this repository (no /root/reference): python tests/golden/make_band_cfg1.py
"""
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
from oracle import oracle_reconstruct_sequence  # noqa: E402
from paper_2507_14046_b200 import workloads as W  # noqa: E402
from paper_2507_14046_b200.priornet import sample_noise_input  # noqa: E402

OUT = Path(__file__).resolve().parent


def main(threads=(2, 4, 8)):
    gq = np.load(OUT / "seq_cfg1.npz")
    spec = W.CONFIGS["cfg1"]
    wl = W.make_workload(spec, seed=0, frames=4)
    z = sample_noise_input(wl.grid, 0, spec.in_channels, 0.1).values
    out = {"threads": np.array(threads)}
    for t in threads:
        torch.set_num_threads(t)
        band = oracle_reconstruct_sequence(spec.channels, spec.in_channels, z, wl.matrix.values,
                                           wl.matrix.columns_q(), [f.values for f in wl.voltages.frames],
                                           gq["theta0"], tuple(gq["output_map"]), 2000, 100, 100, 1e-3)
        out[f"values_t{t}"] = band["columns"].astype(np.float32)
        print("threads", t, "final data", [float(band["traces"][f"frame_{i}"][-1][2]) for i in range(1, 5)], flush=True)
    np.savez_compressed(OUT / "seq_cfg1_band.npz", **out)


if __name__ == "__main__":
    main(tuple(int(a) for a in sys.argv[1:]) or (2, 4, 8))
