"""The network object of the drop-in surface (`pkg/src/d2ip/priornet.py:285-317`).

``build_model(cfg, grid_shape)`` returns a ``DeviceModel``: the parameters of the
reference's ``FastResUNet3D`` (``NetworkConfig``) or of the BASELINE config
ResUNet (``ResUNetConfig``) in ONE flat fp32 CUDA buffer laid out in the
reference's ``state_dict`` order (``param_schema``), with ``state_dict()`` /
``load_state_dict()`` / ``parameters()`` views carrying the reference names and
shapes, and a forward that runs the engine's sm_100a kernels (the same ones a
DIP iteration runs; no CPU path). ``extract_parameters`` / ``load_parameters`` /
``forward_volume`` keep the reference's signatures.

The model is an inference object: training happens in `_FrameOptimizer`
(graph-replayed iterations on the engine), so calling it does not record an
autograd graph.
"""

from __future__ import annotations

from collections import OrderedDict

import numpy as np
import torch

from .priornet import NetworkConfig, NoiseInput, ParameterState, ResUNetConfig, param_schema, state_from_flat


class DeviceModel:
    """GPU-resident parameters + forward of one network configuration."""

    def __init__(self, cfg, grid_shape=None):
        if not isinstance(cfg, (NetworkConfig, ResUNetConfig)):
            raise TypeError(f"unknown network config {type(cfg).__name__}")
        from .engine import require_cuda

        require_cuda()
        self.cfg = cfg
        self.grid_shape = None if grid_shape is None else tuple(int(x) for x in grid_shape)
        self.schema = param_schema(cfg)
        n = sum(e.numel for e in self.schema)
        self._flat = torch.zeros(n, dtype=torch.float32, device="cuda")
        self._views = OrderedDict()
        o = 0
        for e in self.schema:
            self._views[e.name] = self._flat[o:o + e.numel].view(e.shape)
            o += e.numel
        self._net = None
        self.training = True

    # -- torch.nn.Module-like surface -------------------------------------------
    def state_dict(self) -> "OrderedDict[str, torch.Tensor]":
        return OrderedDict((k, v) for k, v in self._views.items())

    def load_state_dict(self, state: dict) -> None:
        missing = [k for k in self._views if k not in state]
        extra = [k for k in state if k not in self._views]
        if missing or extra:
            raise RuntimeError(f"state_dict mismatch: missing {missing[:4]}, unexpected {extra[:4]}")
        with torch.no_grad():
            for k, v in self._views.items():
                t = torch.as_tensor(state[k])
                if tuple(t.shape) != tuple(v.shape):
                    raise RuntimeError(f"size mismatch for {k}: {tuple(t.shape)} vs {tuple(v.shape)}")
                v.copy_(t.to(device="cuda", dtype=torch.float32))

    def parameters(self):
        return iter(self._views.values())

    def named_parameters(self):
        return iter(self._views.items())

    def flat(self) -> torch.Tensor:
        """The flat fp32 parameter buffer (reference state_dict order) on the GPU."""
        return self._flat

    def eval(self):
        self.training = False
        return self

    def train(self, mode: bool = True):
        self.training = mode
        return self

    # -- forward ----------------------------------------------------------------
    def _engine(self, shape):
        from .engine import DeviceNet

        if self._net is not None and self._net_shape == shape:
            return self._net
        mask = np.ones(shape, dtype=bool)
        # forward-only binding: the data term is never evaluated (one zero measurement row)
        dn = DeviceNet(self.cfg, shape, 1, mask, output_map=(0.0, 1.0), precision="fp32", max_iters=1)
        dn.set_J(torch.zeros((1, dn.Vp), dtype=torch.float32, device="cuda"))
        self._net, self._net_shape = dn, shape
        return dn

    def __call__(self, z) -> torch.Tensor:
        return self.forward(z)

    def forward(self, z) -> torch.Tensor:
        """sigmoid network output, an (R, C, P) fp32 CUDA tensor, for the fixed input z
        ((R, C, P) noise for FastResUNet3D, (C_z, R, C, P) for the config ResUNet),
        as `FastResUNet3D.forward` (`priornet.py:217-232`)."""
        zv = z.detach().cpu().numpy() if torch.is_tensor(z) else np.asarray(z)
        shape = tuple(int(x) for x in zv.shape[-3:])
        if self.grid_shape is not None and shape != self.grid_shape:
            raise ValueError(f"input grid {shape} does not match the model's {self.grid_shape}")
        dn = self._engine(shape)
        dn.set_noise(zv)
        dn.theta[0].copy_(self._flat)
        dn.forward(with_loss=False)
        return dn.sig[0].reshape(shape).clone()


def build_model(cfg, grid_shape=None) -> DeviceModel:
    """`build_model` (`priornet.py:285-286`): the network of `cfg`, GPU-backed."""
    return DeviceModel(cfg, grid_shape)


def extract_parameters(model, iteration_counter: int, provenance: str) -> ParameterState:
    """`extract_parameters` (`priornet.py:296-301`): detached CPU clones in state_dict order."""
    if isinstance(model, DeviceModel):
        return state_from_flat(model.flat(), model.schema, iteration_counter, provenance)
    return ParameterState({k: v.detach().clone() for k, v in model.state_dict().items()}, iteration_counter,
                          provenance)


def load_parameters(model, state: ParameterState):
    """`load_parameters` (`priornet.py:304-307`)."""
    model.load_state_dict(dict(state.tensors))
    return model


def forward_volume(cfg, state: ParameterState, noise: NoiseInput) -> np.ndarray:
    """`forward_volume` (`priornet.py:310-317`): the network output for one parameter set
    and noise input, as an (R, C, P) float64 array."""
    model = build_model(cfg, noise.shape)
    load_parameters(model, state)
    model.eval()
    out = model(noise.values)
    return out.cpu().numpy().astype(np.float64)
