"""4D-TV configuration, frame history and the TV functionals
(`pkg/src/d2ip/regularizers.py:31-140`).

Inside the DIP loop the TV value/gradient is computed by the engine's fused
``tv_k`` kernel with the history resident in HBM. The
standalone ``spatial_tv`` / ``temporal_tv`` / ``tv4d`` of the reference's API run
the same kernel through the C ABI (``d2ip_tv4d``): numpy input returns a float,
tensor input a 0-d tensor on the input's device that carries the gradient
w.r.t. ``current`` (computed by the kernel in the same pass) for autograd.
"""

from __future__ import annotations

import math
from dataclasses import dataclass
from typing import Iterable

import numpy as np


@dataclass(frozen=True)
class TVWeights:
    lambda_tv: float = 0.002
    lambda_s: float = 1.0
    lambda_t: float = 0.1
    epsilon: float = 1e-8

    def __post_init__(self):
        if min(self.lambda_tv, self.lambda_s, self.lambda_t) < 0:
            raise ValueError("TV weights must be nonnegative")
        if self.epsilon <= 0:
            raise ValueError("epsilon must be strictly positive")


class FrameHistory:
    """Previously reconstructed volumes of one sequence run, oldest first."""

    def __init__(self, frames: Iterable = ()):
        self._frames = [self._check(f) for f in frames]

    @staticmethod
    def _check(frame):
        if frame.ndim != 3:
            raise ValueError(f"history frames must be 3D volumes, got shape {frame.shape}")
        return frame

    def append(self, frame) -> None:
        if self._frames and tuple(frame.shape) != tuple(self._frames[0].shape):
            raise ValueError("history frames must share one grid shape")
        self._frames.append(self._check(frame))

    @property
    def frames(self) -> list:
        return list(self._frames)

    def __len__(self) -> int:
        return len(self._frames)

    def __iter__(self):
        return iter(self._frames)


def decay_weight(j: int, i: int) -> float:
    """exp(-(i - j)) (`regularizers.py:98-102`)."""
    if not 1 <= j < i:
        raise ValueError(f"need 1 <= j < i, got j={j}, i={i}")
    return math.exp(-(i - j))


# ---------------------------------------------------------------------------
# TV functionals on the device (regularizers.py:86-140)


def _tv_device(current, history, lam_s: float, lam_t: float, eps: float):
    """(value tensor [1], grad [R][C][P]) on the GPU for one volume + history."""
    import torch

    from . import _native as N
    from .engine import _stream_ptr, require_cuda

    require_cuda()
    cur = current.detach().to(device="cuda", dtype=torch.float32).contiguous()
    if cur.ndim != 3:
        raise ValueError(f"expected a 3D volume, got shape {tuple(cur.shape)}")
    R, C, P = (int(x) for x in cur.shape)
    hist = None
    if history:
        hs = []
        for f in history:
            t = f.detach() if torch.is_tensor(f) else torch.as_tensor(np.asarray(f))
            t = t.to(device="cuda", dtype=torch.float32)
            if tuple(t.shape) != (R, C, P):
                raise ValueError("history frame shape does not match the current volume")
            hs.append(t)
        hist = torch.stack(hs).contiguous()
    L = N.lib()
    wsn = int(L.d2ip_tv4d_ws_bytes(R, C, P))
    ws = torch.empty(wsn, dtype=torch.uint8, device="cuda")
    val = torch.empty(1, dtype=torch.float32, device="cuda")
    grad = torch.empty((R, C, P), dtype=torch.float32, device="cuda")
    N.check(L.d2ip_tv4d(N.C.c_void_p(cur.data_ptr()), N.C.c_void_p(hist.data_ptr() if hist is not None else 0),
                        0 if hist is None else hist.shape[0], R, C, P, float(lam_s), float(lam_t), float(eps),
                        N.C.c_void_p(val.data_ptr()), N.C.c_void_p(grad.data_ptr()), N.C.c_void_p(ws.data_ptr()),
                        wsn, N.C.c_void_p(_stream_ptr())), "tv4d")
    return val, grad


def _tv_call(history, current, lam_s, lam_t, eps):
    import torch

    from_numpy = not torch.is_tensor(current)
    if from_numpy:
        vol = np.asarray(current)
        if vol.ndim != 3:
            raise ValueError(f"expected a 3D volume, got shape {vol.shape}")
        val, _ = _tv_device(torch.as_tensor(vol), history, lam_s, lam_t, eps)
        return float(val.item())
    if current.ndim != 3:
        raise ValueError(f"expected a 3D volume, got shape {tuple(current.shape)}")
    return _TVFunction.apply(current, list(history or ()), lam_s, lam_t, eps)


def _make_tv_function():
    import torch

    class TVFunction(torch.autograd.Function):
        @staticmethod
        def forward(ctx, current, history, lam_s, lam_t, eps):
            val, grad = _tv_device(current, history, lam_s, lam_t, eps)
            ctx.save_for_backward(grad)
            ctx.dev, ctx.dtype = current.device, current.dtype
            return val.reshape(()).to(device=current.device, dtype=current.dtype)

        @staticmethod
        def backward(ctx, g):
            (grad,) = ctx.saved_tensors
            return (grad * g.to(grad.device)).to(device=ctx.dev, dtype=ctx.dtype), None, None, None, None

    return TVFunction


class _LazyTV:
    fn = None

    def apply(self, *a):
        if _LazyTV.fn is None:
            _LazyTV.fn = _make_tv_function()
        return _LazyTV.fn.apply(*a)


_TVFunction = _LazyTV()


def spatial_tv(volume, epsilon: float = 1e-8):
    """Isotropic spatial TV of one (R, C, P) volume (`regularizers.py:86-95`)."""
    return _tv_call([], volume, 1.0, 0.0, epsilon)


def temporal_tv(history, current, epsilon: float = 1e-8):
    """Decay-weighted temporal variation against the history (`regularizers.py:105-131`);
    0 for an empty history."""
    frames = list(history)
    import torch

    if not frames:
        if torch.is_tensor(current):
            if current.ndim != 3:
                raise ValueError(f"expected a 3D volume, got shape {tuple(current.shape)}")
            return torch.zeros((), dtype=current.dtype, device=current.device)
        if np.asarray(current).ndim != 3:
            raise ValueError(f"expected a 3D volume, got shape {np.asarray(current).shape}")
        return 0.0
    return _tv_call(frames, current, 0.0, 1.0, epsilon)


def tv4d(history, current, weights: TVWeights):
    """lambda_s * spatial_tv + lambda_t * temporal_tv (`regularizers.py:134-140`)."""
    return _tv_call(list(history), current, weights.lambda_s, weights.lambda_t, weights.epsilon)
