"""Per-frame quality of the long (300/60/60) sequence vs the reference golden (diagnostic)."""
import sys
import numpy as np
sys.path.insert(0, ".")
sys.path.insert(0, "tests")
from conftest import GOLDEN
from oracle.metrics import misfit, mssim
from paper_2507_14046_b200 import RunConfig, TVWeights, reconstruct_sequence
from paper_2507_14046_b200 import workloads as W

gq = np.load(GOLDEN / "seq_long.npz")
spec = W.small_spec()
wl = W.make_workload(spec, seed=0)
prec = sys.argv[1] if len(sys.argv) > 1 else "tf32"
cfg = RunConfig(iters_warm=300, iters_first=60, iters_next=60, learning_rate=1e-3, tv_weights=TVWeights(lambda_tv=0.0),
                seed=1, network=spec.network(), output_map=tuple(gq["output_map"]), data_norm="l2sq", precision=prec)
res = reconstruct_sequence(wl.matrix, wl.voltages, cfg, wl.grid)
R = wl.grid.shape
qc = wl.matrix.columns_q()
vol = lambda col: np.transpose(col.reshape(R[2], R[0], R[1]), (1, 2, 0))  # noqa: E731
for i in range(res.sequence.n_frames):
    a, b, c = vol(res.sequence.values[:, i]), vol(gq["values"][:, i]), vol(gq["band_values"][:, i])
    dv = wl.voltages.frames[i].values
    print(i, "mssim_vs_truth dev %.3f ref %.3f band %.3f" % (mssim(a, wl.truth[i]), mssim(b, wl.truth[i]), mssim(c, wl.truth[i])),
          "misfit dev %.3f ref %.3f band %.3f" % tuple(misfit(wl.matrix.values, qc, v, dv) for v in (a, b, c)))
