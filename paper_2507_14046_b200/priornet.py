"""Network definition, parameters and checkpoints of the drop-in surface.

The GPU engine runs the canonical config ResUNet of SURVEY §7.1 — the
reference topology of `pkg/src/d2ip/priornet.py:183-232` with SE, ASPP and
attention gates removed, dense 3x3x3 convolutions (`_conv3(depthwise=False)`,
`priornet.py:111-117`), `ChannelLayerNorm` (`priornet.py:96-108`) and
LeakyReLU(0.2) in place of SiLU:

    stem  = conv3(Cz -> c0) -> CLN -> act                     (cf. N:199-201)
    enc   = (L-1) x ResConv3d(c[l-1] -> c[l], stride 2)       (cf. N:134-148, 203-205)
    neck  = ResConv3d(c[L-1] -> c[L-1])                       (cf. N:206)
    dec   = (L-1) x [trilinear x2 -> cat(up, skip) -> ResConv3d(c[l+1]+c[l] -> c[l])]
    tail  = conv3(c0 -> 1) -> sigmoid                          (cf. N:215, 231)

Parameter names, shapes (OIDHW) and order are exactly what the equivalent
``nn.Module`` tree's ``state_dict()`` yields, so ``ParameterState`` checksums
(`priornet.py:259-264`) and checkpoints (`priornet.py:324-355`) interoperate
with the reference. Initialisation restates `_kaiming_reset`
(`priornet.py:267-282`): one CPU ``torch.Generator`` seeded once, N(0, 2/fan_in)
per convolution weight in module order, zero biases, identity norms.

The parameters live on the GPU as one flat fp32 buffer in this same order and
layout; export to a ``ParameterState`` is a split + reshape, never a
re-layout, so TPP hand-off checksums are bit-exact.
"""

from __future__ import annotations

import hashlib
import json
from dataclasses import dataclass, field

import numpy as np
import torch

from .errors import FormatError

CHECKPOINT_SCHEMA = 1
PROVENANCES = ("kaiming_init", "upws", "tpp")


@dataclass(frozen=True)
class NetworkConfig:
    """The reference backbone's config (`priornet.py:37-53`).

    The reference-exact FastResUNet3D (SE / ASPP / attention / depthwise) is a
    SURVEY §8(f) "next" item; the engine raises ``NotImplementedError`` for it.
    """

    base_channels: int = 8
    depth: int = 3
    aspp_dilations: tuple = (1, 2, 4)
    use_depthwise: bool = True
    seed: int = 0

    def __post_init__(self):
        if self.depth != 3:
            raise ValueError("the backbone is fixed at three encoder stages")
        if self.base_channels < 4:
            raise ValueError(f"base_channels must be >= 4, got {self.base_channels}")
        dil = tuple(self.aspp_dilations)
        if not dil or any(b <= a for a, b in zip(dil, dil[1:])):
            raise ValueError("aspp_dilations must be nonempty and strictly increasing")
        object.__setattr__(self, "aspp_dilations", dil)


@dataclass(frozen=True)
class ResUNetConfig:
    """Canonical L-level residual U-Net of the BASELINE configs.

    ``channels`` = (c0, ..., c_{L-1}); ``in_channels`` = C_z; the fixed input is
    ``noise_scale * U[0, 1)`` with C_z channels. The reference-config fields
    (``base_channels``/``depth``/``aspp_dilations``/``use_depthwise``) are
    derived so `RunConfig.to_json` (`pipeline.py:108-131`) keeps working.
    """

    channels: tuple = (8, 16)
    in_channels: int = 4
    negative_slope: float = 0.2
    noise_scale: float = 0.1
    seed: int = 0

    def __post_init__(self):
        ch = tuple(int(c) for c in self.channels)
        if len(ch) < 2:
            raise ValueError("a residual U-Net needs at least 2 levels")
        if any(c < 4 or c % 4 for c in ch):
            raise ValueError(f"channels must be positive multiples of 4, got {ch}")
        if self.in_channels < 1:
            raise ValueError("in_channels must be >= 1")
        object.__setattr__(self, "channels", ch)

    @property
    def levels(self) -> int:
        return len(self.channels)

    @property
    def base_channels(self) -> int:
        return self.channels[0]

    @property
    def depth(self) -> int:
        return self.levels - 1

    @property
    def aspp_dilations(self) -> tuple:
        return ()

    @property
    def use_depthwise(self) -> bool:
        return False

    def to_json(self) -> dict:
        return {
            "channels": list(self.channels),
            "in_channels": self.in_channels,
            "negative_slope": self.negative_slope,
            "noise_scale": self.noise_scale,
            "seed": self.seed,
            # reference-config view (pipeline.py:119-126)
            "base_channels": self.base_channels,
            "depth": self.depth,
            "aspp_dilations": [],
            "use_depthwise": False,
        }

    @classmethod
    def from_json(cls, doc: dict) -> "ResUNetConfig":
        return cls(
            channels=tuple(doc["channels"]),
            in_channels=int(doc["in_channels"]),
            negative_slope=float(doc.get("negative_slope", 0.2)),
            noise_scale=float(doc.get("noise_scale", 0.1)),
            seed=int(doc.get("seed", 0)),
        )


def config_hash(cfg) -> str:
    """sha256 of the config without its seed (`priornet.py:56-66`)."""
    if isinstance(cfg, ResUNetConfig):
        doc = cfg.to_json()
        doc.pop("seed")
    else:
        doc = {
            "base_channels": cfg.base_channels,
            "depth": cfg.depth,
            "aspp_dilations": list(cfg.aspp_dilations),
            "use_depthwise": cfg.use_depthwise,
        }
    return hashlib.sha256(json.dumps(doc, sort_keys=True).encode()).hexdigest()[:16]


# ---------------------------------------------------------------------------
# Parameter schema: (name, shape, kind) in state_dict order.


@dataclass(frozen=True)
class ParamEntry:
    name: str
    shape: tuple
    kind: str  # "conv_w" | "conv_b" | "norm_w" | "norm_b"
    fan_in: int = 0

    @property
    def numel(self) -> int:
        return int(np.prod(self.shape))


def _conv(prefix, cin, cout, k):
    return [
        ParamEntry(f"{prefix}.weight", (cout, cin, k, k, k), "conv_w", cin * k * k * k),
        ParamEntry(f"{prefix}.bias", (cout,), "conv_b"),
    ]


def _norm(prefix, c):
    return [ParamEntry(f"{prefix}.weight", (c,), "norm_w"), ParamEntry(f"{prefix}.bias", (c,), "norm_b")]


def _resconv(prefix, cin, cout):
    # registration order of ResConv3d (priornet.py:139-143)
    return (
        _conv(f"{prefix}.conv1", cin, cout, 3)
        + _norm(f"{prefix}.norm1", cout)
        + _conv(f"{prefix}.conv2", cout, cout, 3)
        + _norm(f"{prefix}.norm2", cout)
        + _conv(f"{prefix}.skip", cin, cout, 1)
    )


def _conv3(prefix, cin, cout, depthwise):
    # `_conv3` (priornet.py:111-117): depthwise 3^3 (groups=cin) + pointwise 1^3, or dense 3^3
    if depthwise:
        return _conv(f"{prefix}.0", 1, cin, 3) + _conv(f"{prefix}.1", cin, cout, 1)
    return _conv(prefix, cin, cout, 3)


def _resconv_ref(prefix, cin, cout, depthwise):
    # ResConv3d (priornet.py:134-148)
    return (
        _conv3(f"{prefix}.conv1", cin, cout, depthwise)
        + _norm(f"{prefix}.norm1", cout)
        + _conv3(f"{prefix}.conv2", cout, cout, depthwise)
        + _norm(f"{prefix}.norm2", cout)
        + _conv(f"{prefix}.skip", cin, cout, 1)
    )


def fast_resunet_schema(cfg: NetworkConfig) -> list[ParamEntry]:
    """State-dict order of FastResUNet3D (priornet.py:183-215)."""
    b = cfg.base_channels
    ch = [b, 2 * b, 4 * b, 8 * b]
    dw = cfg.use_depthwise
    out = _conv("stem.0", 1, b, 3) + _norm("stem.1", b)
    for i in range(3):  # SqueezeExcite (priornet.py:120-131)
        hid = max(ch[i] // 4, 1)
        out += _conv(f"enc_se.{i}.fc1", ch[i], hid, 1) + _conv(f"enc_se.{i}.fc2", hid, ch[i], 1)
    for i in range(3):
        out += _resconv_ref(f"enc_block.{i}", ch[i], ch[i + 1], dw)
    for j, _d in enumerate(cfg.aspp_dilations):  # ASPP3d (priornet.py:151-164)
        out += _conv(f"bottleneck.branches.{j}", ch[3], ch[3], 3)
    out += _conv("bottleneck.project", ch[3] * len(cfg.aspp_dilations), ch[3], 1) + _norm("bottleneck.norm", ch[3])
    for j, i in enumerate(reversed(range(3))):  # AttentionGate3d (priornet.py:167-180)
        inter = max(ch[i] // 2, 4)
        out += (_conv(f"dec_att.{j}.key", ch[i], inter, 1) + _conv(f"dec_att.{j}.query", ch[i + 1], inter, 1)
                + _conv(f"dec_att.{j}.score", inter, 1, 1))
    for j, i in enumerate(reversed(range(3))):
        out += _resconv_ref(f"dec_block.{j}", ch[i + 1] + ch[i], ch[i], dw)
    out += _conv("tail", b, 1, 3)
    return out


def param_schema(cfg) -> list[ParamEntry]:
    """State-dict order of the network (module registration order,
    `priornet.py:199-215`; the config ResUNet drops SE/ASPP/attention)."""
    if isinstance(cfg, NetworkConfig):
        return fast_resunet_schema(cfg)
    if not isinstance(cfg, ResUNetConfig):
        raise TypeError(f"unknown network config {type(cfg).__name__}")
    c = cfg.channels
    L = len(c)
    out = _conv("stem.0", cfg.in_channels, c[0], 3) + _norm("stem.1", c[0])
    for i in range(1, L):
        out += _resconv(f"enc_block.{i - 1}", c[i - 1], c[i])
    out += _resconv("bottleneck", c[L - 1], c[L - 1])
    for j, lvl in enumerate(reversed(range(L - 1))):
        out += _resconv(f"dec_block.{j}", c[lvl + 1] + c[lvl], c[lvl])
    out += _conv("tail", c[0], 1, 3)
    return out


def param_offsets(schema) -> dict[str, tuple[int, tuple]]:
    offs, o = {}, 0
    for e in schema:
        offs[e.name] = (o, e.shape)
        o += e.numel
    return offs


def count_parameters(cfg) -> int:
    return sum(e.numel for e in param_schema(cfg))


# ---------------------------------------------------------------------------


@dataclass
class ParameterState:
    """Named parameter tensors handed between stages (`priornet.py:235-264`)."""

    tensors: dict
    iteration_counter: int = 0
    provenance: str = "kaiming_init"
    # host-side caches (not part of the value): the sha256 of the tensors, and
    # the flat fp32 buffer the state was exported from (same bytes)
    _sha: str | None = field(default=None, repr=False, compare=False)
    _flat: torch.Tensor | None = field(default=None, repr=False, compare=False)

    def __post_init__(self):
        if self.provenance not in PROVENANCES:
            raise ValueError(f"unknown provenance {self.provenance!r}")
        if self._flat is not None:  # exported from one flat buffer: one vectorised finiteness check
            if not bool(torch.isfinite(self._flat).all()):
                for name, t in self.tensors.items():
                    if not torch.isfinite(t).all():
                        raise ValueError(f"parameter tensor {name} contains non-finite values")
            return
        for name, t in self.tensors.items():
            if not torch.isfinite(t).all():
                raise ValueError(f"parameter tensor {name} contains non-finite values")

    def clone(self, provenance=None, iteration_counter=None) -> "ParameterState":
        flat = self._flat.clone() if self._flat is not None else None
        if flat is not None:  # the clones are views of one new flat buffer, like the original
            tensors, o = {}, 0
            for k, v in self.tensors.items():
                tensors[k] = flat[o:o + v.numel()].view(v.shape)
                o += v.numel()
        else:
            tensors = {k: v.detach().clone() for k, v in self.tensors.items()}
        return ParameterState(
            tensors=tensors,
            iteration_counter=self.iteration_counter if iteration_counter is None else iteration_counter,
            provenance=self.provenance if provenance is None else provenance,
            _sha=self._sha, _flat=flat,
        )

    def checksum(self) -> str:
        if self._sha is not None:
            return self._sha
        digest = hashlib.sha256()
        for name, t in self.tensors.items():
            digest.update(name.encode())
            digest.update(t.detach().cpu().contiguous().numpy().tobytes())
        # cached: the tensors are detached clones handed between stages, never mutated in place
        object.__setattr__(self, "_sha", digest.hexdigest())
        return self._sha

    def flat(self, schema=None) -> torch.Tensor:
        """Concatenate into the engine's flat fp32 layout (state-dict order)."""
        names = [e.name for e in schema] if schema is not None else list(self.tensors)
        if self._flat is not None and names == list(self.tensors):
            return self._flat
        return torch.cat([self.tensors[n].detach().reshape(-1).to(torch.float32).cpu() for n in names])


def state_from_flat(flat: torch.Tensor, schema, iteration_counter=0, provenance="kaiming_init") -> ParameterState:
    """Tensors are views of one private host copy of `flat` (one D2H copy, one
    finiteness check, and `flat()` can hand the buffer back without a cat)."""
    flat = flat.detach().to("cpu", torch.float32).contiguous().clone()
    tensors, o = {}, 0
    for e in schema:
        tensors[e.name] = flat[o:o + e.numel].view(e.shape)
        o += e.numel
    if o != flat.numel():
        raise ValueError(f"flat buffer has {flat.numel()} values, schema needs {o}")
    return ParameterState(tensors, iteration_counter, provenance, _flat=flat)


def kaiming_flat(cfg, seed: int | None = None) -> torch.Tensor:
    """Flat θ0 restating `_kaiming_reset` (`priornet.py:267-282`)."""
    schema = param_schema(cfg)
    gen = torch.Generator().manual_seed(cfg.seed if seed is None else seed)
    parts = []
    for e in schema:
        if e.kind == "conv_w":
            t = torch.empty(e.shape, dtype=torch.float32)
            t.normal_(0.0, (2.0 / e.fan_in) ** 0.5, generator=gen)
        elif e.kind == "norm_w":
            t = torch.ones(e.shape, dtype=torch.float32)
        else:
            t = torch.zeros(e.shape, dtype=torch.float32)
        parts.append(t.reshape(-1))
    return torch.cat(parts)


def init_parameters(cfg) -> ParameterState:
    """Freshly seeded parameters (`priornet.py:289-293`)."""
    schema = param_schema(cfg)
    return state_from_flat(kaiming_flat(cfg), schema, 0, "kaiming_init")


# ---------------------------------------------------------------------------


@dataclass(frozen=True)
class NoiseInput:
    """Fixed network input. 3D values = the reference's 1-channel U[0,1) noise
    (`priornet.py:69-93`); 4D values (C_z, R, C, P) = the config input."""

    values: np.ndarray
    seed: int

    def __post_init__(self):
        vals = np.ascontiguousarray(self.values, dtype=np.float64)
        if vals.ndim not in (3, 4):
            raise ValueError(f"noise input must be 3D or (C, R, C, P), got shape {vals.shape}")
        vals.setflags(write=False)
        object.__setattr__(self, "values", vals)

    @property
    def shape(self) -> tuple[int, int, int]:
        return tuple(self.values.shape[-3:])

    @property
    def channels(self) -> int:
        return 1 if self.values.ndim == 3 else self.values.shape[0]

    def sha256(self) -> str:
        return hashlib.sha256(self.values.tobytes()).hexdigest()


def sample_noise_input(grid, seed: int, channels: int = 1, scale: float = 1.0) -> NoiseInput:
    """`sample_noise_input` (`priornet.py:91-93`); with ``channels``/``scale``
    the config input ``scale * U[0,1)`` of shape (C_z, R, C, P)."""
    rng = np.random.default_rng(seed)
    shape = tuple(grid.shape)
    if channels == 1 and scale == 1.0:
        return NoiseInput(rng.random(shape), seed)
    return NoiseInput(scale * rng.random((channels,) + shape), seed)


def noise_for(cfg, grid, seed: int) -> NoiseInput:
    if isinstance(cfg, ResUNetConfig):
        return sample_noise_input(grid, seed, cfg.in_channels, cfg.noise_scale)
    return sample_noise_input(grid, seed)


# ---------------------------------------------------------------------------


def save_checkpoint(path, state: ParameterState, cfg, noise_sha256=None) -> None:
    """`priornet.py:324-340`."""
    torch.save(
        {
            "schema_version": CHECKPOINT_SCHEMA,
            "config_hash": config_hash(cfg),
            "provenance": state.provenance,
            "iteration_counter": state.iteration_counter,
            "noise_sha256": noise_sha256,
            "tensors": {k: v.detach().cpu() for k, v in state.tensors.items()},
        },
        path,
    )


def load_checkpoint(path, cfg) -> ParameterState:
    """`priornet.py:343-355`."""
    doc = torch.load(path, weights_only=True)
    if doc.get("schema_version") != CHECKPOINT_SCHEMA:
        raise FormatError(f"unsupported checkpoint schema in {path}")
    if doc.get("config_hash") != config_hash(cfg):
        raise FormatError(f"checkpoint {path} was written for a different network configuration")
    return ParameterState(
        tensors=doc["tensors"],
        iteration_counter=int(doc["iteration_counter"]),
        provenance=doc["provenance"],
    )
