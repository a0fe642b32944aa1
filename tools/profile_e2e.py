"""cProfile of one cfg1 reconstruct_sequence (the bench's e2e call)."""
import cProfile
import pstats
import sys
import time

sys.path.insert(0, ".")
import torch  # noqa: E402

from paper_2507_14046_b200 import reconstruct_sequence  # noqa: E402
from paper_2507_14046_b200 import workloads as W  # noqa: E402
from paper_2507_14046_b200.forward import MaskedSensitivity, VoltageSequence  # noqa: E402

spec = W.CONFIGS["cfg1"]
wl = W.make_workload(spec, seed=0, frames=20)
cfg = W.run_config_for(spec, wl.output_map, seed=0, precision="tf32")
matrix = MaskedSensitivity(wl.matrix.values, wl.matrix.mask)
volts = VoltageSequence(wl.voltages.frames[:20])
reconstruct_sequence(matrix, VoltageSequence(wl.voltages.frames[:2]), cfg, wl.grid)  # warm
torch.cuda.synchronize()
pr = cProfile.Profile()
t0 = time.perf_counter()
pr.enable()
res = reconstruct_sequence(matrix, volts, cfg, wl.grid)
torch.cuda.synchronize()
pr.disable()
print("wall", time.perf_counter() - t0)
pstats.Stats(pr).sort_stats("cumulative").print_stats(30)
