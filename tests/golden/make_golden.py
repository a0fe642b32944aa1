"""Generate the golden fixtures by running the REAL reference package.

Run in the build container only (needs /root/reference):
    python tests/golden/make_golden.py

The reference cannot express the BASELINE config networks, so
the config ResUNet is injected into it exactly as SURVEY §8(c) verified:
  * the residual blocks ARE the reference's own `ResConv3d`
    (`pkg/src/d2ip/priornet.py:134-148`, dense convs `use_depthwise=False`),
    with the module-level `F.silu` it calls rebound to LeakyReLU(0.2) for the
    duration of the run, and the reference `ChannelLayerNorm` (:96-108);
  * only the U-Net wiring (stem / encoder / bottleneck / trilinear-up + cat
    decoder / tail) is written here;
  * `d2ip.pipeline.build_model`, `d2ip.priornet.build_model` and
    `d2ip.pipeline.sample_noise_input` are patched so the reference's
    unmodified `_FrameOptimizer`, `_kaiming_reset`, `init_parameters`,
    `upws_pretrain` and `reconstruct_sequence` run it;
  * J is passed as the reference's dense `SensitivityMatrix` with zero
    columns outside the cylinder mask.
Inputs come from `paper_2507_14046_b200.workloads` (seeded); their sha256 are
stored so the tests can prove the harness still generates the same arrays.
"""

from __future__ import annotations

import hashlib
import sys
import types
from dataclasses import dataclass, replace
from pathlib import Path

import numpy as np
import torch
import torch.nn.functional as TF
from torch import nn

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, "/root/reference/pkg/src")

import d2ip.pipeline as P  # noqa: E402
import d2ip.priornet as N  # noqa: E402
from d2ip.forward import SensitivityMatrix, VoltageFrame, VoltageSequence  # noqa: E402
from d2ip.regularizers import FrameHistory, TVWeights  # noqa: E402

from paper_2507_14046_b200 import workloads as W  # noqa: E402
from paper_2507_14046_b200.geometry import vectorize  # noqa: E402
from paper_2507_14046_b200.priornet import sample_noise_input  # noqa: E402

OUT = Path(__file__).resolve().parent
SLOPE = 0.2


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


# -- LeakyReLU in place of SiLU inside the reference ResConv3d --------------
_shim = types.ModuleType("F_leaky")
for _k in dir(TF):
    setattr(_shim, _k, getattr(TF, _k))
_shim.silu = lambda x: TF.leaky_relu(x, SLOPE)
N.F = _shim


@dataclass(frozen=True)
class GoldenNetCfg:
    channels: tuple
    in_channels: int
    seed: int = 0
    base_channels: int = 8
    depth: int = 2
    aspp_dilations: tuple = ()
    use_depthwise: bool = False


class GoldenResUNet(nn.Module):
    def __init__(self, cfg: GoldenNetCfg, grid_shape=None):
        super().__init__()
        c = list(cfg.channels)
        L = len(c)
        self.stem = nn.Sequential(nn.Conv3d(cfg.in_channels, c[0], 3, padding=1),
                                  N.ChannelLayerNorm(c[0]), nn.LeakyReLU(SLOPE))
        self.enc_block = nn.ModuleList(N.ResConv3d(c[i - 1], c[i], stride=2, depthwise=False)
                                       for i in range(1, L))
        self.bottleneck = N.ResConv3d(c[L - 1], c[L - 1], depthwise=False)
        self.dec_block = nn.ModuleList(N.ResConv3d(c[i + 1] + c[i], c[i], depthwise=False)
                                       for i in reversed(range(L - 1)))
        self.tail = nn.Conv3d(c[0], 1, 3, padding=1)

    def forward(self, z):
        x = self.stem(z[None])
        skips = []
        for b in self.enc_block:
            skips.append(x)
            x = b(x)
        x = self.bottleneck(x)
        for b, s in zip(self.dec_block, reversed(skips)):
            x = TF.interpolate(x, size=s.shape[2:], mode="trilinear", align_corners=False)
            x = b(torch.cat([x, s], dim=1))
        return torch.sigmoid(self.tail(x))[0, 0]


def _build(cfg, grid_shape=None):
    return GoldenResUNet(cfg, grid_shape)


N.build_model = _build
P.build_model = _build


class _Noise:
    def __init__(self, ni):
        self.values = ni.values
        self.shape = ni.shape
        self._sha = ni.sha256()

    def sha256(self):
        return self._sha


def flat_state(state) -> np.ndarray:
    return torch.cat([t.reshape(-1) for t in state.tensors.values()]).numpy().astype(np.float32)


def dense_matrix(masked) -> SensitivityMatrix:
    d = masked.dense()
    return SensitivityMatrix(d.values, True, True, masked.grid_ref, masked.protocol_ref)


def grads_of(runner, theta, dv, history, cfg):
    N.load_parameters(runner.model, theta)
    runner.cfg = cfg
    runner.model.zero_grad(set_to_none=True)
    dv_t = torch.as_tensor(np.asarray(dv), dtype=torch.float32)
    total, data, reg, mapped = runner.loss_terms(dv_t, history)
    total.backward()
    g = torch.cat([p.grad.reshape(-1) for p in runner.model.parameters()]).numpy().astype(np.float32)
    return float(total), float(data), float(reg), g


def case_cfg0():
    spec = W.CONFIGS["cfg0"]
    wl = W.make_workload(spec, seed=0)
    grid = wl.grid
    noise = sample_noise_input(grid, 0, spec.in_channels, 0.1)
    net = GoldenNetCfg(spec.channels, spec.in_channels, seed=1)
    cfg = P.RunConfig(iters_warm=300, iters_first=300, iters_next=300, learning_rate=1e-3,
                      tv_weights=TVWeights(lambda_tv=0.0), seed=0, network=net,
                      output_map=wl.output_map, data_norm="l2sq")
    matrix = dense_matrix(wl.matrix)
    dv = wl.voltages.frames[0].values
    theta0 = N.init_parameters(net)
    runner = P._FrameOptimizer(cfg, matrix, _Noise(noise))
    out = {"theta0": flat_state(theta0), "theta0_sha": theta0.checksum(),
           "J_sha": sha(wl.matrix.values), "dv": dv, "dv_sha": sha(dv), "z_sha": noise.sha256(),
           "output_map": np.array(wl.output_map)}
    # step-1 loss and gradients, three loss variants
    t, d, r, g = grads_of(runner, theta0, dv, FrameHistory(), cfg)
    out.update(l2sq_total=t, l2sq_data=d, l2sq_grads=g)
    cfg_l2 = replace(cfg, data_norm="l2")
    t, d, r, g = grads_of(runner, theta0, dv, FrameHistory(), cfg_l2)
    out.update(l2_total=t, l2_data=d, l2_grads=g)
    rng = np.random.default_rng(7)
    hist = [torch.as_tensor(rng.normal(scale=0.05, size=grid.shape), dtype=torch.float32) for _ in range(2)]
    cfg_tv = replace(cfg, tv_weights=TVWeights(), data_norm="l2")
    t, d, r, g = grads_of(runner, theta0, dv, FrameHistory(hist), cfg_tv)
    out.update(tv_total=t, tv_data=d, tv_reg=r, tv_grads=g, tv_history=np.stack([h.numpy() for h in hist]))
    runner.cfg = cfg
    # theta after 1 and 10 Adam steps; trace of 10
    for k in (1, 10):
        vol, mapped, th, tr = runner.optimize(theta0, dv, FrameHistory(), k, frame_label=0)
        out[f"theta{k}"] = flat_state(th)
        out[f"trace{k}"] = np.array([[r.iteration, r.data_term, r.total] for r in tr.records])
        out[f"volume{k}"] = vol
    # the full 300-iteration single-frame run (BASELINE cfg0)
    torch.set_num_threads(1)
    vol, mapped, th, tr = runner.optimize(theta0, dv, FrameHistory(), 300, frame_label=0)
    out["theta300"] = flat_state(th)
    out["trace300"] = np.array([[r.iteration, r.data_term, r.total] for r in tr.records])
    out["volume300"] = vol
    np.savez_compressed(OUT / "cfg0_step.npz", **out)
    print("cfg0: step-1 data", out["l2sq_data"], "final data", out["trace300"][-1, 1])


def case_sequence():
    spec = W.small_spec()
    wl = W.make_workload(spec, seed=0)
    grid = wl.grid
    net = GoldenNetCfg(spec.channels, spec.in_channels, seed=0)
    noise = sample_noise_input(grid, 1, spec.in_channels, 0.1)
    P.sample_noise_input = lambda g, s: _Noise(sample_noise_input(grid, s, spec.in_channels, 0.1))
    cfg = P.RunConfig(iters_warm=12, iters_first=6, iters_next=4, learning_rate=1e-3,
                      tv_weights=TVWeights(lambda_tv=0.0), seed=1, network=net,
                      output_map=wl.output_map, data_norm="l2sq")
    matrix = dense_matrix(wl.matrix)
    volts = VoltageSequence([VoltageFrame(f.values, f.frame_index) for f in wl.voltages.frames])
    res = P.reconstruct_sequence(matrix, volts, cfg, grid)
    out = {"J_sha": sha(wl.matrix.values), "z_sha": noise.sha256(),
           "output_map": np.array(wl.output_map),
           "provenance": np.array([s.provenance for s in res.provenance_chain]),
           "iterations": np.array([f.iterations for f in res.frame_records]),
           "values": res.sequence.values,
           "theta_final": flat_state(res.states["final"]),
           "theta_warm": flat_state(res.states["warm"]),
           "theta0": flat_state(res.states["init"])}
    for key, tr in res.traces.items():
        out[f"trace_{key}"] = np.array([[r.iteration, r.data_term, r.total] for r in tr.records])
    # with TV on (reference default weights) and l2 norm, 3 frames
    cfg_tv = replace(cfg, tv_weights=TVWeights(), data_norm="l2")
    volts3 = VoltageSequence(volts.frames[:3])
    res_tv = P.reconstruct_sequence(matrix, volts3, cfg_tv, grid)
    out["tv_values"] = res_tv.sequence.values
    for key, tr in res_tv.traces.items():
        out[f"tvtrace_{key}"] = np.array([[r.iteration, r.data_term, r.total] for r in tr.records])
    np.savez_compressed(OUT / "seq_mini.npz", **out)
    print("sequence:", list(out["provenance"]), list(out["iterations"]))


def case_sequence_long():
    """Converged budgets (300 UPWS / 60 / 60, 4 frames): the end-to-end bar
    (MSSIM >= 0.99, data misfit within 2%) is judged on these volumes."""
    spec = W.small_spec()
    wl = W.make_workload(spec, seed=0)
    grid = wl.grid
    net = GoldenNetCfg(spec.channels, spec.in_channels, seed=0)
    P.sample_noise_input = lambda g, s: _Noise(sample_noise_input(grid, s, spec.in_channels, 0.1))
    cfg = P.RunConfig(iters_warm=300, iters_first=60, iters_next=60, learning_rate=1e-3,
                      tv_weights=TVWeights(lambda_tv=0.0), seed=1, network=net,
                      output_map=wl.output_map, data_norm="l2sq")
    matrix = dense_matrix(wl.matrix)
    volts = VoltageSequence([VoltageFrame(f.values, f.frame_index) for f in wl.voltages.frames])
    res = P.reconstruct_sequence(matrix, volts, cfg, grid)
    out = {"values": res.sequence.values, "output_map": np.array(wl.output_map),
           "iterations": np.array([f.iterations for f in res.frame_records])}
    for key, tr in res.traces.items():
        out[f"trace_{key}"] = np.array([[r.iteration, r.data_term, r.total] for r in tr.records])
    # Natural fp32 variability band: the same algorithm with only the
    # summation order of J.sigma changed (compact masked J, CPU oracle). Long
    # DIP trajectories are chaotic, so this is the yardstick for end-to-end
    # agreement.
    sys.path.insert(0, str(ROOT))
    from oracle import oracle_reconstruct_sequence
    theta0 = flat_state(res.states["init"])
    band = oracle_reconstruct_sequence(spec.channels, spec.in_channels,
                                       sample_noise_input(grid, 1, spec.in_channels, 0.1).values,
                                       wl.matrix.values, wl.matrix.columns_q(),
                                       [f.values for f in wl.voltages.frames], theta0, wl.output_map,
                                       300, 60, 60, 1e-3)
    out["band_values"] = band["columns"]
    np.savez_compressed(OUT / "seq_long.npz", **out)
    print("long sequence: final data terms", [float(out[f"trace_frame_{i}"][-1, 1]) for i in range(1, 5)])


def case_level4():
    """A 4-level injected net (channels 4/8/16/32 on a 16x16x16 grid, the cfg2 / cfg4
    topology at a fixture-sized width): step-1 loss + gradients and theta after 5 Adam
    steps, pinning the oracle / engine at L = 4 (SURVEY §7.1 restatement of
    priornet.py:183-232). theta0 is stored by checksum (kaiming, bit-reproducible)."""
    spec = W.small_spec(name="l4", grid=(16, 16, 16), channels=(4, 8, 16, 32), in_channels=4,
                        rings=(0.3, 0.7), frames=1)
    wl = W.make_workload(spec, seed=2)
    grid = wl.grid
    noise = sample_noise_input(grid, 2, spec.in_channels, 0.1)
    net = GoldenNetCfg(spec.channels, spec.in_channels, seed=3, depth=4)
    cfg = P.RunConfig(iters_warm=5, iters_first=5, iters_next=5, learning_rate=1e-3,
                      tv_weights=TVWeights(lambda_tv=0.0), seed=2, network=net,
                      output_map=wl.output_map, data_norm="l2sq")
    matrix = dense_matrix(wl.matrix)
    dv = wl.voltages.frames[0].values
    theta0 = N.init_parameters(net)
    runner = P._FrameOptimizer(cfg, matrix, _Noise(noise))
    out = {"theta0_sha": theta0.checksum(), "J_sha": sha(wl.matrix.values),
           "dv": dv, "z_sha": noise.sha256(), "output_map": np.array(wl.output_map),
           "channels": np.array(spec.channels), "grid": np.array(grid.shape), "net_seed": 3}
    t, d, r, g = grads_of(runner, theta0, dv, FrameHistory(), cfg)
    out.update(l2sq_total=t, l2sq_data=d, l2sq_grads=g)
    for k in (5,):
        vol, mapped, th, tr = runner.optimize(theta0, dv, FrameHistory(), k, frame_label=0)
        out[f"theta{k}"] = flat_state(th)
        out[f"trace{k}"] = np.array([[r.iteration, r.data_term, r.total] for r in tr.records])
    np.savez_compressed(OUT / "level4.npz", **out)
    print("level4: params", out["l2sq_grads"].size, "step-1 data", d)


def case_joint():
    """cfg4's joint warm-start check: the reference's `upws_pretrain`
    with dv0 = the mean of F frames (one shared Z), 10 iterations. The joint loss
    sum_f ||J sigma - dv_f||^2 has F times this gradient; Adam is scale-invariant
    up to eps, so the engine's joint run must land on the same theta."""
    spec = W.small_spec(grid=(8, 8, 8), channels=(8, 16), in_channels=4, rings=(0.5,), frames=4)
    wl = W.make_workload(spec, seed=0)
    grid = wl.grid
    noise = sample_noise_input(grid, 0, 4, 0.1)
    net = GoldenNetCfg(spec.channels, spec.in_channels, seed=1)
    cfg = P.RunConfig(iters_warm=10, iters_first=10, iters_next=10, learning_rate=1e-3,
                      tv_weights=TVWeights(lambda_tv=0.0), seed=0, network=net,
                      output_map=wl.output_map, data_norm="l2sq")
    dvs = np.stack([f.values for f in wl.voltages.frames])
    theta0 = N.init_parameters(net)
    state, trace = P.upws_pretrain(dense_matrix(wl.matrix), dvs.mean(0), _Noise(noise), cfg, theta_init=theta0)
    np.savez_compressed(OUT / "joint_upws.npz", dvs=dvs, theta0=flat_state(theta0), theta10=flat_state(state),
                        output_map=np.array(wl.output_map),
                        trace=np.array([[r.iteration, r.data_term, r.total] for r in trace.records]))
    print("joint: final data", trace.records[-1].data_term)


def case_cfg1_sequence(frames: int = 4):
    """BASELINE cfg1 budgets on the cfg1 workload: UPWS 2,000 on frame 1, then frame 1
    (100) and a TPP chain of frames 2..`frames` (100 each), run by the reference with
    its dense operator (all host threads: `serial=False`). The oracle with the compact
    masked J (same algorithm, only J.sigma's fp32 summation order changed) gives the
    natural variability band the GPU result is judged against."""
    spec = W.CONFIGS["cfg1"]
    wl = W.make_workload(spec, seed=0, frames=frames)
    grid = wl.grid
    net = GoldenNetCfg(spec.channels, spec.in_channels, seed=0)
    P.sample_noise_input = lambda g, s: _Noise(sample_noise_input(grid, s, spec.in_channels, 0.1))
    cfg = P.RunConfig(iters_warm=2000, iters_first=100, iters_next=100, learning_rate=1e-3,
                      tv_weights=TVWeights(lambda_tv=0.0), seed=0, network=net,
                      output_map=wl.output_map, data_norm="l2sq", serial=False)
    torch.set_num_threads(max(1, __import__("os").cpu_count()))
    matrix = dense_matrix(wl.matrix)
    volts = VoltageSequence([VoltageFrame(f.values, f.frame_index) for f in wl.voltages.frames])
    res = P.reconstruct_sequence(matrix, volts, cfg, grid)
    out = {"values": res.sequence.values.astype(np.float32), "output_map": np.array(wl.output_map),
           "iterations": np.array([f.iterations for f in res.frame_records]),
           "theta0": flat_state(res.states["init"]), "J_sha": sha(wl.matrix.values)}
    for key, tr in res.traces.items():
        out[f"trace_{key}"] = np.array([r.data_term for r in tr.records], dtype=np.float32)
    from oracle import oracle_reconstruct_sequence
    band = oracle_reconstruct_sequence(spec.channels, spec.in_channels,
                                       sample_noise_input(grid, 0, spec.in_channels, 0.1).values,
                                       wl.matrix.values, wl.matrix.columns_q(),
                                       [f.values for f in wl.voltages.frames], out["theta0"], wl.output_map,
                                       2000, 100, 100, 1e-3)
    out["band_values"] = band["columns"].astype(np.float32)
    for key, tr in band["traces"].items():
        out[f"band_trace_{key}"] = np.array([r[2] for r in tr], dtype=np.float32)
    np.savez_compressed(OUT / "seq_cfg1.npz", **out)
    print("cfg1 sequence: final data", [float(out[f"trace_frame_{i}"][-1]) for i in range(1, frames + 1)],
          "band", [float(out[f"band_trace_frame_{i}"][-1]) for i in range(1, frames + 1)])


if __name__ == "__main__":
    torch.set_num_threads(1)
    which = sys.argv[1:] or ["cfg0", "sequence", "long", "level4", "joint", "cfg1seq"]
    if "level4" in which:
        case_level4()
    if "joint" in which:
        case_joint()
    if "cfg1seq" in which:
        case_cfg1_sequence()
    if "cfg0" in which:
        case_cfg0()
    if "sequence" in which:
        case_sequence()
    if "long" in which:
        case_sequence_long()
