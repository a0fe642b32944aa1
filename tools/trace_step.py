"""Concurrent timeline of one eager cfg1 DIP iteration (debug).

Records CUDA events around every launch (d2ip_trace_begin / d2ip_trace_dump),
prints each launch as start / end / stream / kernel, then per-stream busy time
and the span. Events between launches defeat PDL overlap, so the span reads a
little longer than the graph-replayed bench step.

    python tools/trace_step.py [--workload cfg1] [--out gpurun_out/trace.txt]
"""
import argparse
import ctypes as C
import sys

sys.path.insert(0, ".")
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2507_14046_b200 import _native as N  # noqa: E402
from paper_2507_14046_b200 import workloads as W  # noqa: E402
from paper_2507_14046_b200.engine import DeviceNet  # noqa: E402
from paper_2507_14046_b200.priornet import kaiming_flat, sample_noise_input  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="cfg1")
ap.add_argument("--out", default=None)
ap.add_argument("--reps", type=int, default=3)
args = ap.parse_args()

spec = W.CONFIGS[args.workload]
wl = W.make_workload(spec, seed=0, frames=2)
net = spec.network(seed=1)
dn = DeviceNet(net, wl.grid.shape, wl.matrix.n_measurements, wl.matrix.mask, data_norm="l2sq",
               output_map=wl.output_map, lr=spec.learning_rate, precision=spec.precision, max_iters=64)
dn.set_noise(sample_noise_input(wl.grid, 0, spec.in_channels, 0.1).values)
dn.set_J_host(wl.matrix.values)
dn.set_theta(kaiming_flat(net))
dn.set_dv(wl.voltages.frames[0].values)
dn.reset_frame()
for _ in range(5):
    dn.run(1, graph=False)
torch.cuda.synchronize()
L = N.lib()
buf = C.create_string_buffer(1 << 20)
best = None
for _ in range(args.reps):
    L.d2ip_trace_begin()
    dn.run(1, graph=False)
    L.d2ip_trace_dump(buf, len(buf))
    rows = []
    for ln in buf.value.decode().splitlines():
        s, e, st, name = ln.split(" ", 3)
        rows.append((float(s), float(e), st, name))
    span = max(r[1] for r in rows)
    if best is None or span < best[0]:
        best = (span, rows)
span, rows = best
streams = {}
for r in rows:
    streams.setdefault(r[2], len(streams))
lines = [f"span {span:.1f} us, {len(rows)} launches, {len(streams)} streams"]
for s, e, st, name in sorted(rows):
    lines.append(f"{s:8.1f} {e:8.1f} {e - s:7.1f}  s{streams[st]}  {name[:90]}")
for st, i in streams.items():
    busy = sum(e - s for s, e, t, _ in rows if t == st)
    last = max(e for s, e, t, _ in rows if t == st)
    lines.append(f"stream s{i}: busy {busy:.1f} us, last end {last:.1f} us")
txt = "\n".join(lines)
print(txt)
if args.out:
    open(args.out, "w").write(txt + "\n")
