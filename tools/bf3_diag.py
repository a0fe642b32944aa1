"""3xbf16 vs 3xTF32 forward: engine-vs-engine differences (debug). Run twice with D2IP_BF3_MASK."""
import sys, os
sys.path.insert(0, ".")
import numpy as np, torch
from paper_2507_14046_b200 import workloads as W
from paper_2507_14046_b200.engine import DeviceNet
from paper_2507_14046_b200.priornet import kaiming_flat, sample_noise_input
name = sys.argv[1]
full = W.CONFIGS[name]
spec = W.WorkloadSpec(name + "-r", (32, 32, 16), full.ring_heights, full.channels, full.in_channels, 1, 1, 1, 1)
wl = W.make_workload(spec, seed=0, frames=1)
net = spec.network(seed=1)
noise = sample_noise_input(wl.grid, 0, spec.in_channels, 0.1)
theta = kaiming_flat(net)
dv = wl.voltages.frames[0].values
dn = DeviceNet(net, wl.grid.shape, wl.matrix.n_measurements, wl.matrix.mask, output_map=wl.output_map, precision="tf32", max_iters=4)
dn.set_noise(noise.values); dn.set_J_host(wl.matrix.values); dn.set_theta(theta); dn.set_dv(dv)
out = []
for rep in range(2):
    dn.reset_frame(); dn.grads(); torch.cuda.synchronize()
    out.append((dn.grad[0].clone(), dn.sig[0].clone(), float(dn.trace_host(0, 1)[0, 0])))
print("repeat bitwise equal:", torch.equal(out[0][0], out[1][0]), torch.equal(out[0][1], out[1][1]))
np.savez(sys.argv[2], grad=out[0][0].cpu().numpy(), sig=out[0][1].cpu().numpy(), data=out[0][2])
if len(sys.argv) > 3:
    o = np.load(sys.argv[3])
    g, s = out[0][0].cpu().numpy(), out[0][1].cpu().numpy()
    print("vs other: grad rel", np.linalg.norm(g - o["grad"]) / np.linalg.norm(o["grad"]),
          "sig rel", np.linalg.norm(s - o["sig"]) / np.linalg.norm(o["sig"]), "max abs sig", np.abs(s - o["sig"]).max(),
          "data", out[0][2], float(o["data"]))
