"""Multi-GPU partitioning of the DIP step.

* Single sequences (cfg0/1/2) do not shard: the TPP chain is sequential
  (`pkg/src/d2ip/pipeline.py:523-557`); N GPUs run N independent replicas.
* Independent sequences (BASELINE cfg3) shard: `shard()` gives each rank an
  even, contiguous slice of the sequence indices; a rank runs its slice in
  lockstep as ONE batched engine (per-sequence θ, Z, J: the convolutions are
  grouped over the batch, J·Σ is a batched GEMV over distinct J) and results
  are gathered once at the end — no collective inside the loop.
* The joint warm-start of cfg4 optimises one network against F frames at once
  (loss Σ_f ||Jσ − Δv_f||²). Frames are partitioned over ranks; every
  iteration each rank computes the gradient of its frames' loss on the engine,
  the flat gradient buffers are summed with one all-reduce (NCCL over NVLink
  in production, gloo in the CPU tests), and every rank applies the identical
  Adam update — θ stays bitwise identical across ranks.

`joint_upws` only needs an object with ``grads()``, ``adam()`` and a ``grad``
tensor, so the host logic is testable on the CPU with a stand-in model.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch
import torch.distributed as dist


def shard(n_items: int, world: int, rank: int) -> range:
    """Even contiguous partition: the first n % world ranks get one extra."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} / world {world}")
    base, extra = divmod(n_items, world)
    start = rank * base + min(rank, extra)
    return range(start, start + base + (1 if rank < extra else 0))


def world_info():
    if dist.is_available() and dist.is_initialized():
        return dist.get_world_size(), dist.get_rank()
    return 1, 0


def gather_to_root(obj, root: int = 0):
    """Gather one picklable object per rank onto `root` (None elsewhere)."""
    world, rank = world_info()
    if world == 1:
        return [obj]
    out = [None] * world if rank == root else None
    dist.gather_object(obj, out, dst=root)
    return out


def allreduce_grads(grad: torch.Tensor) -> None:
    """Sum the flat gradient buffer over ranks in place (one collective)."""
    world, _ = world_info()
    if world > 1:
        dist.all_reduce(grad, op=dist.ReduceOp.SUM)


def allreduce_status(status: torch.Tensor) -> None:
    """MAX of the per-sequence status words over ranks, in place and in stream order
    (step and history count are equal on every rank; the bad flag becomes "any rank
    saw a non-finite loss", so every rank skips the same Adam updates)."""
    world, _ = world_info()
    if world > 1:
        dist.all_reduce(status, op=dist.ReduceOp.MAX)


def joint_upws(engine, iters: int, data_norm: str = "l2sq", on_step=None, graph: bool = True) -> None:
    """Data-parallel joint warm-start: per iteration grads -> all-reduce(grad, SUM)
    -> all-reduce(status, MAX) -> Adam. `engine.reset_frame()` must have been called
    (fresh optimiser). The summed per-rank gradients are the gradient of the joint
    loss only for the squared norm (sum_f ||J sigma - dv_f||^2); with "l2" each rank's
    sqrt(local sum) would be a different objective, so it is rejected. A non-finite
    loss on any rank freezes theta on every rank and raises NumericalError on every
    rank after the loop (the device never waits on the host inside the loop)."""
    if data_norm != "l2sq":
        raise ValueError(f"joint warm-start needs data_norm='l2sq' (sum of per-frame squared misfits), "
                         f"got {data_norm!r}")
    status = getattr(engine, "status", None)
    for k in range(1, iters + 1):
        engine.grads(graph=graph)  # one CUDA-graph replay of forward + loss + backward
        allreduce_grads(engine.grad)
        if status is not None:
            allreduce_status(status)
        engine.adam()
        if on_step is not None:
            on_step(k)
    if status is not None:
        st = status.cpu().numpy().reshape(-1, 4)
        if (st[:, 1] != 0).any():
            from .errors import NumericalError
            exc = NumericalError(f"non-finite loss in the joint warm-start at iteration {int(st[:, 1].max())}")
            exc.iteration = int(st[:, 1].max())
            raise exc


# ---------------------------------------------------------------------------
# Batched independent sequences on one GPU (the per-rank body of cfg3).


@dataclass
class BatchedResult:
    seeds: list
    volumes: np.ndarray      # [B][T][R][C][P] fp64 (lo + (hi-lo)*sigmoid)
    final_data: np.ndarray   # [B][T] data term at the last iteration of each frame
    iterations: int


def reconstruct_batched(workloads, cfg, seeds, network=None) -> BatchedResult:
    """Run len(workloads) independent sequences in lockstep on one engine with
    the driver logic of `reconstruct_sequence` (UPWS on frame `warm_frame`,
    then the TPP chain; budgets by provenance, fresh Adam per frame)."""
    from .engine import DeviceNet
    from .priornet import kaiming_flat, noise_for

    B = len(workloads)
    if B == 0:
        return BatchedResult([], np.zeros((0,)), np.zeros((0,)), 0)
    wl0 = workloads[0]
    net = network or cfg.network
    T = min(w.voltages.n_frames for w in workloads)
    tv = cfg.tv_weights
    dn = DeviceNet(net, wl0.grid.shape, wl0.matrix.n_measurements, wl0.matrix.mask, batch=B, j_shared=False,
                   data_norm=cfg.data_norm, output_map=cfg.output_map, lr=cfg.learning_rate,
                   betas=cfg.optimizer_betas, precision=cfg.precision,
                   tv=(tv.lambda_tv, tv.lambda_s, tv.lambda_t, tv.epsilon),
                   max_history=max(T - 1, 1) if tv.lambda_tv > 0 else 0,
                   max_iters=max(cfg.iters_warm, cfg.iters_first, cfg.iters_next, 1))
    for b, (w, s) in enumerate(zip(workloads, seeds)):
        if w.matrix.mask.shape != wl0.matrix.mask.shape or not np.array_equal(w.matrix.mask, wl0.matrix.mask):
            raise ValueError("batched sequences must share one voxel mask")
        dn.set_J_host(w.matrix.values, b=b)
        dn.set_noise(noise_for(net, w.grid, s).values, b=b)
        dn.set_theta(kaiming_flat(net, seed=s + 1), b=b)
    vols = np.zeros((B, T) + tuple(wl0.grid.shape))
    final = np.zeros((B, T))
    total = 0

    def stage(iters, frame_idx):
        nonlocal total
        for b, w in enumerate(workloads):
            dn.set_dv(w.voltages.frames[frame_idx].values, b=b)
        dn.reset_frame()
        dn.run(iters)
        total += iters
        st = dn.status_host()
        if np.any(st[:, 1] != 0):
            from .errors import NumericalError
            raise NumericalError(f"non-finite loss in batched sequences {np.flatnonzero(st[:, 1]).tolist()}")

    if not cfg.disable_upws:
        stage(cfg.iters_warm, cfg.warm_frame - 1)
    first = {"kaiming_init": cfg.iters_warm, "upws": cfg.iters_first}["upws" if not cfg.disable_upws else "kaiming_init"]
    # budgets by provenance (pipeline.py:436-441): TPP frames run iters_next,
    # without TPP every frame restarts from the frame-1 initialisation
    budgets = [first] + [first if cfg.disable_tpp else cfg.iters_next] * (T - 1)
    theta1 = dn.theta.clone() if cfg.disable_tpp else None
    for i in range(T):
        if theta1 is not None:
            dn.theta.copy_(theta1)
        stage(budgets[i], i)
        dn.forward(with_loss=False)
        for b in range(B):
            vols[b, i] = dn.volume(b)
            final[b, i] = float(dn.trace_host(b, budgets[i])[budgets[i] - 1, 0]) if budgets[i] else np.nan
        if tv.lambda_tv > 0 and i + 1 < T:
            dn.append_history_from_mapped()
    return BatchedResult(list(seeds), vols, final, total)
