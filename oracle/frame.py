"""The DIP loop restated on the CPU — TEST INFRASTRUCTURE ONLY.

Follows `pkg/src/d2ip/pipeline.py`:
  _vectorize_t            :252-254  q = ((p*R)+r)*C+c, then the mask's columns
  _data_term              :257-263  "l2sq" = sum r^2; "l2" = sqrt (exact zero kept)
  _FrameOptimizer         :266-338  fresh Adam per frame, trace, non-finite check, final forward
  upws / frame / sequence :394-560  budgets by provenance, TPP clone, history append
and 4D-TV `pkg/src/d2ip/regularizers.py:86-140`.
J is the compact masked block (M x V, fp32) with its canonical column indices:
identical arithmetic to the reference's dense operator with zero columns.
"""

from __future__ import annotations

import math
import time

import numpy as np
import torch
import torch.nn.functional as F

from .resunet import build_oracle_net


def _vectorize_t(volume: torch.Tensor) -> torch.Tensor:
    return volume.permute(2, 0, 1).reshape(-1)


def _data_term(residual: torch.Tensor, mode: str) -> torch.Tensor:
    sq = (residual * residual).sum()
    if mode == "l2sq":
        return sq
    if sq.item() == 0.0:
        return sq
    return torch.sqrt(sq)


def _forward_diff(t, dim):
    n = t.shape[dim]
    d = t.narrow(dim, 1, n - 1) - t.narrow(dim, 0, n - 1)
    return torch.cat([d, torch.zeros_like(t.narrow(dim, 0, 1))], dim=dim)


def oracle_tv4d(history, current, lambda_s=1.0, lambda_t=0.1, eps=1e-8):
    """regularizers.py:86-140 (spatial mean + decay-weighted temporal sum)."""
    dr, dc, dp = (_forward_diff(current, d) for d in range(3))
    spatial = torch.sqrt(dr * dr + dc * dc + dp * dp + eps).mean()
    frames = list(history)
    if not frames:
        temporal = torch.zeros((), dtype=current.dtype)
    else:
        i = len(frames) + 1
        total = torch.zeros((), dtype=current.dtype)
        wsum = 0.0
        for k, past in enumerate(frames):
            alpha = math.exp(-(i - (k + 1)))
            diff = current - torch.as_tensor(past, dtype=current.dtype)
            total = total + alpha * torch.sqrt(diff * diff + eps).sum()
            wsum += alpha
        temporal = total / wsum
    return lambda_s * spatial + lambda_t * temporal


class OracleFrameOptimizer:
    """pipeline.py:266-338 for the config ResUNet (or any prebuilt `model`)."""

    def __init__(self, channels, in_channels, z, J, qcols, output_map, lr, betas=(0.9, 0.999),
                 data_norm="l2sq", tv=(0.0, 1.0, 0.1, 1e-8), slope=0.2, record_every=1, model=None):
        # model: a prebuilt network (e.g. oracle.refnet.OracleFastResUNet); else the config ResUNet
        self.model = model if model is not None else build_oracle_net(channels, in_channels, slope)
        self.z = torch.tensor(np.asarray(z), dtype=torch.float32)
        self.J = torch.tensor(np.asarray(J), dtype=torch.float32)
        self.qcols = torch.tensor(np.asarray(qcols), dtype=torch.long)
        self.output_map = tuple(output_map)
        self.lr, self.betas, self.data_norm = lr, tuple(betas), data_norm
        self.tv = tv
        self.record_every = record_every

    def load(self, flat_or_state):
        if isinstance(flat_or_state, dict):
            self.model.load_state_dict({k: torch.as_tensor(v, dtype=torch.float32) for k, v in flat_or_state.items()})
        else:
            flat = torch.as_tensor(flat_or_state, dtype=torch.float32)
            o = 0
            with torch.no_grad():
                for p in self.model.state_dict().values():
                    p.copy_(flat[o:o + p.numel()].reshape(p.shape))
                    o += p.numel()

    def state(self):
        return {k: v.detach().clone() for k, v in self.model.state_dict().items()}

    def flat(self):
        return torch.cat([v.detach().reshape(-1) for v in self.model.state_dict().values()])

    def loss_terms(self, dv, history):
        lo, hi = self.output_map
        out = self.model(self.z)
        mapped = lo + (hi - lo) * out
        residual = dv - self.J @ _vectorize_t(mapped)[self.qcols]
        data = _data_term(residual, self.data_norm)
        lam, ls, lt, eps = self.tv
        reg = lam * oracle_tv4d(history, mapped, ls, lt, eps)
        return data + reg, data, reg, mapped

    def grads(self, dv, history=()):
        """Loss terms and per-parameter gradients of one step (no update)."""
        self.model.zero_grad(set_to_none=True)
        dv_t = torch.as_tensor(np.asarray(dv), dtype=torch.float32)
        total, data, reg, mapped = self.loss_terms(dv_t, history)
        total.backward()
        g = {k: p.grad.detach().clone() for k, p in self.model.named_parameters()}
        return float(total), float(data), float(reg), g, mapped.detach()

    def iterate(self, dv, history, iters, opt=None, frame_label=1):
        """`iters` bodies of the loop at pipeline.py:310-331 (loss terms, finiteness check,
        trace record, zero_grad, backward, Adam step) against a persistent optimiser and
        nothing else -- the bench's CPU arm times exactly one training iteration per step
        (no per-call Adam construction, no final output forward). Returns the optimiser."""
        if opt is None:
            opt = torch.optim.Adam(self.model.parameters(), lr=self.lr, betas=self.betas)
        dv_t = dv if torch.is_tensor(dv) else torch.as_tensor(np.asarray(dv), dtype=torch.float32)
        start = time.perf_counter()
        for k in range(1, iters + 1):
            total, data, reg, _ = self.loss_terms(dv_t, history)
            if not torch.isfinite(total):
                raise FloatingPointError(f"non-finite loss at stage frame={frame_label} iteration={k}")
            _ = (frame_label, k, float(data.detach()), float(torch.as_tensor(reg).detach()),
                 float(total.detach()), time.perf_counter() - start)
            opt.zero_grad(set_to_none=True)
            total.backward()
            opt.step()
        return opt

    def optimize(self, dv, history, iters, frame_label=1):
        opt = torch.optim.Adam(self.model.parameters(), lr=self.lr, betas=self.betas)
        dv_t = torch.as_tensor(np.asarray(dv), dtype=torch.float32)
        trace = []
        start = time.perf_counter()
        for k in range(1, iters + 1):
            total, data, reg, _ = self.loss_terms(dv_t, history)
            if not torch.isfinite(total):
                raise FloatingPointError(f"non-finite loss at stage frame={frame_label} iteration={k}")
            if (k - 1) % self.record_every == 0 or k == iters:
                trace.append((frame_label, k, float(data.detach()), float(torch.as_tensor(reg)), float(total.detach()),
                              time.perf_counter() - start))
            opt.zero_grad(set_to_none=True)
            total.backward()
            opt.step()
        lo, hi = self.output_map
        with torch.no_grad():
            out = self.model(self.z)
            mapped = lo + (hi - lo) * out
        volume = lo + (hi - lo) * out.numpy().astype(np.float64)
        return volume, mapped, trace


def oracle_loss_and_grads(channels, in_channels, z, J, qcols, dv, theta_flat, output_map,
                          data_norm="l2sq", history=(), tv=(0.0, 1.0, 0.1, 1e-8), model=None):
    opt = OracleFrameOptimizer(channels, in_channels, z, J, qcols, output_map, 1e-3,
                               data_norm=data_norm, tv=tv, model=model)
    opt.load(theta_flat)
    return opt.grads(dv, history)


def oracle_reconstruct_sequence(channels, in_channels, z, J, qcols, frames_dv, theta0_flat,
                                output_map, iters_warm, iters_first, iters_next, lr,
                                data_norm="l2sq", tv=(0.0, 1.0, 0.1, 1e-8), warm_frame=1,
                                disable_upws=False, disable_tpp=False, model=None):
    """pipeline.py:444-560 (UPWS -> frame 1 -> TPP chain); returns a dict."""
    runner = OracleFrameOptimizer(channels, in_channels, z, J, qcols, output_map, lr,
                                  data_norm=data_norm, tv=tv, model=model)
    theta0 = torch.as_tensor(theta0_flat, dtype=torch.float32).clone()
    chain = [("kaiming_init", 0)]
    traces = {}
    frame1_init, prov1, ctr1 = theta0, "kaiming_init", 0
    if not disable_upws:
        runner.load(theta0)
        _, _, tr = runner.optimize(frames_dv[warm_frame - 1], [], iters_warm, 0)
        traces["warm"] = tr
        frame1_init, prov1, ctr1 = runner.flat(), "upws", iters_warm
        chain.append(("upws", ctr1))
    budget = {"kaiming_init": iters_warm, "upws": iters_first, "tpp": iters_next}
    history, columns, records = [], [], []
    prev, prev_ctr = None, 0
    for i in range(1, len(frames_dv) + 1):
        if i == 1:
            theta_i, prov, ctr = frame1_init, prov1, ctr1
        elif disable_tpp:
            theta_i, prov, ctr = frame1_init, prov1, ctr1
        else:
            theta_i, prov, ctr = prev, "tpp", prev_ctr
            chain.append(("tpp", ctr))
        iters = budget[prov]
        runner.load(theta_i)
        vol, mapped, tr = runner.optimize(frames_dv[i - 1], history, iters, i)
        traces[f"frame_{i}"] = tr
        history.append(mapped)
        columns.append(np.transpose(vol, (2, 0, 1)).reshape(-1))
        prev, prev_ctr = runner.flat(), ctr + iters
        records.append((i, prov, iters))
    return {"chain": chain, "traces": traces, "columns": np.stack(columns, 1),
            "records": records, "final": prev}
