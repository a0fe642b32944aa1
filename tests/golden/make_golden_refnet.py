"""Golden fixtures of the reference backbone FastResUNet3D, from the REAL,
UNPATCHED reference package (`pkg/src/d2ip`, imported from /root/reference).

Run in the build container only:
    python tests/golden/make_golden_refnet.py

Writes tests/golden/refnet.npz:
  per variant  v in {dw4 (base 4, depthwise), dense4 (base 4, dense 3^3), dw8 (base 8, the
               reference default NetworkConfig)}:
    {v}_theta0_sha     ParameterState.checksum of init_parameters(cfg)
    {v}_l2sq_*         loss terms + flat gradients of step 1 (`loss_terms` + backward)
  dw4 / dense4 only:
    {v}_theta0         flat init_parameters(cfg) (state_dict order)
    {v}_l2_*, {v}_tv_* the "l2" data norm, and "l2" + 4D-TV with a 2-frame history
    {v}_theta1 / theta10, trace10, volume10   `_FrameOptimizer.optimize`
  seq_*        `reconstruct_sequence` (UPWS -> frame 1 -> TPP) with NetworkConfig(base 4)
Inputs come from `paper_2507_14046_b200.workloads` (seeded, 16^3 grid); the
noise is the reference's own `sample_noise_input`; sha256 of every input is
stored so the tests can prove the harness regenerates the same arrays.
"""

from __future__ import annotations

import hashlib
import sys
from dataclasses import replace
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, "/root/reference/pkg/src")

import d2ip.pipeline as P  # noqa: E402
import d2ip.priornet as N  # noqa: E402
from d2ip.forward import SensitivityMatrix, VoltageFrame, VoltageSequence  # noqa: E402
from d2ip.regularizers import FrameHistory, TVWeights  # noqa: E402

from paper_2507_14046_b200 import workloads as W  # noqa: E402

OUT = Path(__file__).resolve().parent
GRID_SEED = 0


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


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


def variant(out, tag, net, wl, noise, full=True):
    grid = wl.grid
    cfg = P.RunConfig(iters_warm=12, iters_first=6, iters_next=4, learning_rate=1e-3,
                      tv_weights=TVWeights(lambda_tv=0.0), seed=0, network=net,
                      output_map=wl.output_map, data_norm="l2sq")
    matrix = dense_matrix(wl.matrix)
    dv = wl.voltages.frames[0].values
    theta0 = N.init_parameters(net)
    runner = P._FrameOptimizer(cfg, matrix, noise)
    if full:
        out[f"{tag}_theta0"] = flat_state(theta0)
    out[f"{tag}_theta0_sha"] = theta0.checksum()
    t, d, r, g = grads_of(runner, theta0, dv, FrameHistory(), cfg)
    out.update({f"{tag}_l2sq_total": t, f"{tag}_l2sq_data": d, f"{tag}_l2sq_grads": g})
    print(tag, "step-1 data", d, "params", g.size)
    if not full:
        return
    t, d, r, g = grads_of(runner, theta0, dv, FrameHistory(), replace(cfg, data_norm="l2"))
    out.update({f"{tag}_l2_total": t, f"{tag}_l2_data": d, f"{tag}_l2_grads": g})
    rng = np.random.default_rng(7)
    hist = [torch.as_tensor(rng.normal(scale=0.05, size=grid.shape), dtype=torch.float32) for _ in range(2)]
    t, d, r, g = grads_of(runner, theta0, dv, FrameHistory(hist),
                          replace(cfg, tv_weights=TVWeights(), data_norm="l2"))
    out.update({f"{tag}_tv_total": t, f"{tag}_tv_data": d, f"{tag}_tv_reg": r, f"{tag}_tv_grads": g})
    out["tv_history"] = np.stack([h.numpy() for h in hist])
    runner.cfg = cfg
    for k in (1, 10):
        vol, mapped, th, tr = runner.optimize(theta0, dv, FrameHistory(), k, frame_label=0)
        out[f"{tag}_theta{k}"] = flat_state(th)
        out[f"{tag}_trace{k}"] = np.array([[r.iteration, r.data_term, r.total] for r in tr.records])
        out[f"{tag}_volume{k}"] = vol


def main():
    torch.set_num_threads(1)
    spec = W.small_spec()
    wl = W.make_workload(spec, seed=0)
    grid = wl.grid
    noise = N.sample_noise_input(grid, GRID_SEED)
    out = {"J_sha": sha(wl.matrix.values), "dv": wl.voltages.frames[0].values,
           "dv_sha": sha(wl.voltages.frames[0].values), "z": noise.values.astype(np.float32),
           "z_sha": noise.sha256(), "output_map": np.array(wl.output_map)}
    variant(out, "dw4", N.NetworkConfig(base_channels=4, use_depthwise=True, seed=1), wl, noise)
    variant(out, "dense4", N.NetworkConfig(base_channels=4, use_depthwise=False, seed=1), wl, noise)
    variant(out, "dw8", N.NetworkConfig(seed=1), wl, noise, full=False)
    # the whole driver (RunConfig.seed -> noise / init seeds inside the reference)
    net = N.NetworkConfig(base_channels=4, seed=0)
    cfg = P.RunConfig(iters_warm=12, iters_first=6, iters_next=4, learning_rate=1e-3,
                      tv_weights=TVWeights(lambda_tv=0.0), seed=1, network=net,
                      output_map=wl.output_map, data_norm="l2sq")
    volts = VoltageSequence([VoltageFrame(f.values, f.frame_index) for f in wl.voltages.frames])
    res = P.reconstruct_sequence(dense_matrix(wl.matrix), volts, cfg, grid)
    out["seq_values"] = res.sequence.values
    out["seq_provenance"] = np.array([s.provenance for s in res.provenance_chain])
    out["seq_iterations"] = np.array([f.iterations for f in res.frame_records])
    out["seq_theta0"] = flat_state(res.states["init"])
    out["seq_theta_warm"] = flat_state(res.states["warm"])
    out["seq_theta_final"] = flat_state(res.states["final"])
    for key, tr in res.traces.items():
        out[f"seq_trace_{key}"] = np.array([[r.iteration, r.data_term, r.total] for r in tr.records])
    np.savez_compressed(OUT / "refnet.npz", **out)
    print("sequence:", list(out["seq_provenance"]), list(out["seq_iterations"]))


if __name__ == "__main__":
    main()
