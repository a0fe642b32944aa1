import sys, os
sys.path.insert(0, ".")
import numpy as np, torch
from oracle import oracle_loss_and_grads
from paper_2507_14046_b200 import workloads as W
from paper_2507_14046_b200.engine import DeviceNet
from paper_2507_14046_b200.priornet import kaiming_flat, sample_noise_input, param_schema
torch.set_num_threads(16)
name, prec = sys.argv[1], sys.argv[2]
full = W.CONFIGS[name]
grid = tuple(int(v) for v in sys.argv[3].split("x")) if len(sys.argv) > 3 else (32, 32, 16)
spec = W.WorkloadSpec(name + "-r", grid, full.ring_heights, full.channels, full.in_channels, 1, 1, 1, 1)
wl = W.make_workload(spec, seed=0, frames=1)
net = spec.network(seed=1)
noise = sample_noise_input(wl.grid, 0, spec.in_channels, 0.1)
theta = kaiming_flat(net)
dv = wl.voltages.frames[0].values
_, data_ref, _, g_ref, _ = oracle_loss_and_grads(spec.channels, spec.in_channels, noise.values, wl.matrix.values,
                                                 wl.matrix.columns_q(), dv, theta, wl.output_map)
dn = DeviceNet(net, wl.grid.shape, wl.matrix.n_measurements, wl.matrix.mask, output_map=wl.output_map, precision=prec, max_iters=4)
dn.set_noise(noise.values); dn.set_J_host(wl.matrix.values); dn.set_theta(theta); dn.set_dv(dv)
dn.reset_frame(); dn.grads(); torch.cuda.synchronize()
gd = dn.grad[0].cpu().numpy()
flat = torch.cat([v.reshape(-1) for v in g_ref.values()]).numpy()
tag = " ".join(f"{k}={v}" for k, v in os.environ.items() if k.startswith("D2IP_"))
print(f"[{tag}] {name} {prec} data rel {abs(float(dn.trace_host(0,1)[0,0])-data_ref)/data_ref:.2e} grad rel {np.linalg.norm(gd - flat) / np.linalg.norm(flat):.3e}")
o = 0
worst = []
for e in param_schema(net):
    r = g_ref[e.name].reshape(-1).numpy()
    err = np.linalg.norm(gd[o:o + e.numel] - r) / max(np.linalg.norm(r), 1e-30)
    worst.append((err, e.name, np.linalg.norm(r)))
    o += e.numel
for err, n, g in sorted(worst, reverse=True)[:6]:
    print(f"    {n:28s} |g|={g:.3e} rel={err:.3e}")
