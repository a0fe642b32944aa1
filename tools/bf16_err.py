"""Per-tensor gradient error of the bf16 engine path vs the CPU oracle (debug)."""
import sys
sys.path.insert(0, ".")
import numpy as np, torch
from oracle import oracle_loss_and_grads
from paper_2507_14046_b200 import workloads as W
from paper_2507_14046_b200.engine import DeviceNet
from paper_2507_14046_b200.priornet import kaiming_flat, sample_noise_input, param_schema
for shape in sys.argv[1:] or ["mini", "cfg1"]:
    spec = W.small_spec() if shape == "mini" else W.CONFIGS[shape]
    wl = W.make_workload(spec, seed=0, frames=1)
    net = spec.network(seed=1)
    noise = sample_noise_input(wl.grid, 0, spec.in_channels, 0.1)
    theta = kaiming_flat(net)
    dv = wl.voltages.frames[0].values
    _, data_ref, _, g_ref, _ = oracle_loss_and_grads(spec.channels, spec.in_channels, noise.values, wl.matrix.values,
                                                     wl.matrix.columns_q(), dv, theta, wl.output_map)
    for prec in ["bf16"]:
        dn = DeviceNet(net, wl.grid.shape, wl.matrix.n_measurements, wl.matrix.mask, output_map=wl.output_map,
                       precision=prec, max_iters=4)
        dn.set_noise(noise.values); dn.set_J_host(wl.matrix.values); dn.set_theta(theta); dn.set_dv(dv)
        dn.reset_frame(); dn.grads(); torch.cuda.synchronize()
        gd = dn.grad[0].cpu().numpy()
        flat = torch.cat([v.reshape(-1) for v in g_ref.values()]).numpy()
        print(shape, prec, "data", float(dn.trace_host(0, 1)[0, 0]), data_ref, "grad rel", np.linalg.norm(gd - flat) / np.linalg.norm(flat))
        o = 0
        for e in param_schema(net):
            r = g_ref[e.name].reshape(-1).numpy()
            err = np.linalg.norm(gd[o:o + e.numel] - r) / max(np.linalg.norm(r), 1e-30)
            print(f"   {e.name:28s} n={e.numel:7d} |g|={np.linalg.norm(r):.3e} rel={err:.3e}")
            o += e.numel
