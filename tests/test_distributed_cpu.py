"""Multi-process host logic on the CPU (gloo, world size 2): the cfg3 sequence
sharding and gather, and the cfg4 joint-UPWS gradient all-reduce, with a CPU
stand-in for the engine (the device kernels are covered by -m gpu tests)."""

import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2507_14046_b200.distributed import gather_to_root, joint_upws, shard


def test_shard_partitions_evenly():
    for n in (0, 1, 7, 64):
        for world in (1, 2, 3, 8):
            parts = [shard(n, world, r) for r in range(world)]
            flat = [i for p in parts for i in p]
            assert flat == list(range(n))
            assert max(len(p) for p in parts) - min(len(p) for p in parts) <= 1
    with pytest.raises(ValueError):
        shard(4, 2, 2)


class LstsqEngine:
    """Stand-in with the engine's joint-UPWS interface: loss sum_f |A x - d_f|^2
    over this rank's frames, Adam exactly as the K7 kernel / torch.optim.Adam."""

    def __init__(self, A, frames, x0, lr=1e-2):
        self.A, self.frames = A, frames
        self.theta = x0.clone()
        self.grad = torch.zeros_like(x0)
        self.m = torch.zeros_like(x0)
        self.v = torch.zeros_like(x0)
        self.t = 0
        self.lr = lr
        self.status = torch.zeros((1, 4), dtype=torch.int32)  # [step, bad iteration, n_hist, -]

    def grads(self, graph=False):
        r = sum(self.A @ self.theta - d for d in self.frames) if self.frames else torch.zeros(self.A.shape[0])
        self.grad.copy_(2 * self.A.T @ r)
        self.status[0, 0] += 1
        if not torch.isfinite(r).all() and self.status[0, 1] == 0:
            self.status[0, 1] = int(self.status[0, 0])

    def adam(self):
        if self.status[0, 1] != 0:
            return
        self.t += 1
        b1, b2, eps = 0.9, 0.999, 1e-8
        self.m.lerp_(self.grad, 1 - b1)
        self.v.mul_(b2).addcmul_(self.grad, self.grad, value=1 - b2)
        step = self.lr / (1 - b1 ** self.t)
        denom = (self.v.sqrt() / (1 - b2 ** self.t) ** 0.5).add_(eps)
        self.theta.addcdiv_(self.m, denom, value=-step)


def _problem():
    g = torch.Generator().manual_seed(0)
    A = torch.randn(12, 5, generator=g, dtype=torch.float64)
    frames = [torch.randn(12, generator=g, dtype=torch.float64) for _ in range(4)]
    x0 = torch.zeros(5, dtype=torch.float64)
    return A, frames, x0


def _worker_nan(rank, world, port, out):
    """rank 1 sees a non-finite frame: every rank must freeze theta and raise."""
    from paper_2507_14046_b200.errors import NumericalError
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        A, frames, x0 = _problem()
        mine = [frames[i] for i in shard(len(frames), world, rank)]
        if rank == 1:
            mine[0] = mine[0].clone()
            mine[0][3] = float("nan")
        eng = LstsqEngine(A, mine, x0)
        try:
            joint_upws(eng, 5)
            out.put((rank, "no error", None))
        except NumericalError as e:
            out.put((rank, "raised", (e.iteration, eng.theta.tolist())))
    finally:
        dist.destroy_process_group()


def _worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        A, frames, x0 = _problem()
        mine = [frames[i] for i in shard(len(frames), world, rank)]
        eng = LstsqEngine(A, mine, x0)
        joint_upws(eng, 25)
        got = gather_to_root(eng.theta.tolist())
        seqs = gather_to_root(list(shard(64, world, rank)))
        if rank == 0:
            out.put((got, seqs))
    finally:
        dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_joint_upws_allreduce_matches_single_process():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    thetas, seqs = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    # every rank holds the identical θ
    assert thetas[0] == thetas[1]
    # and it equals one process optimising the joint loss over all frames
    A, frames, x0 = _problem()
    ref = LstsqEngine(A, frames, x0)
    joint_upws(ref, 25)
    assert torch.allclose(torch.tensor(thetas[0], dtype=torch.float64), ref.theta, rtol=1e-12, atol=1e-12)
    # the 64 cfg3 sequences are split 32/32 and gathered in rank order
    assert [i for s in seqs for i in s] == list(range(64))


def test_joint_upws_rejects_l2_norm():
    A, frames, x0 = _problem()
    with pytest.raises(ValueError):
        joint_upws(LstsqEngine(A, frames, x0), 1, data_norm="l2")


def test_joint_upws_nonfinite_raises_on_every_rank():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker_nan, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert [r[1] for r in res] == ["raised", "raised"]
    # both ranks report the same iteration and kept the identical (initial) theta
    assert res[0][2] == res[1][2]
    assert res[0][2][0] == 1 and res[0][2][1] == [0.0] * 5
