"""Config ResUNet restated in CPU PyTorch — TEST INFRASTRUCTURE ONLY.

Topology: SURVEY §7.1, following `pkg/src/d2ip/priornet.py`:
  ChannelLayerNorm  priornet.py:96-108   (per-voxel LayerNorm over channels, eps 1e-5)
  ResConv3d         priornet.py:134-148  (conv1 -> norm1 -> act -> conv2 -> norm2, 1^3 skip, add, act)
  FastResUNet3D     priornet.py:183-232  (stem, encoder blocks, bottleneck, trilinear-up + cat
                                          decoder blocks, tail conv -> sigmoid), minus SE/ASPP/attention
  _kaiming_reset    priornet.py:267-282
with LeakyReLU(negative_slope) instead of SiLU (BASELINE.json shared convention (d)).
"""

from __future__ import annotations

import torch
import torch.nn.functional as F
from torch import nn


class ChannelLayerNorm(nn.Module):
    """priornet.py:96-108."""

    def __init__(self, channels: int, eps: float = 1e-5):
        super().__init__()
        self.weight = nn.Parameter(torch.ones(channels))
        self.bias = nn.Parameter(torch.zeros(channels))
        self.eps = eps

    def forward(self, x):
        xp = x.movedim(1, -1)
        xp = F.layer_norm(xp, (xp.shape[-1],), self.weight, self.bias, self.eps)
        return xp.movedim(-1, 1)


class ResConv(nn.Module):
    """priornet.py:134-148 with dense 3^3 convs (use_depthwise=False, :117)."""

    def __init__(self, cin, cout, stride, slope, norm_cls=ChannelLayerNorm):
        super().__init__()
        self.conv1 = nn.Conv3d(cin, cout, 3, stride=stride, padding=1)
        self.norm1 = norm_cls(cout)
        self.conv2 = nn.Conv3d(cout, cout, 3, padding=1)
        self.norm2 = norm_cls(cout)
        self.skip = nn.Conv3d(cin, cout, 1, stride=stride)
        self.slope = slope

    def forward(self, x):
        h = F.leaky_relu(self.norm1(self.conv1(x)), self.slope)
        h = self.norm2(self.conv2(h))
        return F.leaky_relu(h + self.skip(x), self.slope)


class ConfigResUNet(nn.Module):
    """Canonical L-level residual U-Net; forward returns the (R, C, P) volume
    for a 4D (C_z, R, C, P) or 5D input, as `_vectorize_t` expects (pipeline.py:252)."""

    def __init__(self, channels, in_channels, slope=0.2, norm_cls=ChannelLayerNorm):
        super().__init__()
        c = list(channels)
        L = len(c)
        self.stem = nn.Sequential(nn.Conv3d(in_channels, c[0], 3, padding=1), norm_cls(c[0]),
                                  nn.LeakyReLU(slope))
        self.enc_block = nn.ModuleList(ResConv(c[i - 1], c[i], 2, slope, norm_cls) for i in range(1, L))
        self.bottleneck = ResConv(c[L - 1], c[L - 1], 1, slope, norm_cls)
        self.dec_block = nn.ModuleList(
            ResConv(c[i + 1] + c[i], c[i], 1, slope, norm_cls) for i in reversed(range(L - 1))
        )
        self.tail = nn.Conv3d(c[0], 1, 3, padding=1)

    def forward(self, z):
        x = z[None] if z.ndim == 4 else z
        squeeze = z.ndim == 4
        x = self.stem(x)
        skips = []
        for block in self.enc_block:
            skips.append(x)
            x = block(x)
        x = self.bottleneck(x)
        for block, s in zip(self.dec_block, reversed(skips)):
            x = F.interpolate(x, size=s.shape[2:], mode="trilinear", align_corners=False)
            x = block(torch.cat([x, s], dim=1))
        out = torch.sigmoid(self.tail(x))
        return out[0, 0] if squeeze else out[:, 0]


def kaiming_reset(model: nn.Module, seed: int, norm_cls=ChannelLayerNorm) -> None:
    """priornet.py:267-282."""
    gen = torch.Generator().manual_seed(seed)
    with torch.no_grad():
        for module in model.modules():
            if isinstance(module, nn.Conv3d):
                fan_in = module.in_channels // module.groups
                for k in module.kernel_size:
                    fan_in *= k
                module.weight.normal_(0.0, (2.0 / fan_in) ** 0.5, generator=gen)
                if module.bias is not None:
                    module.bias.zero_()
            elif isinstance(module, norm_cls):
                module.weight.fill_(1.0)
                module.bias.zero_()


def build_oracle_net(channels, in_channels, slope=0.2, seed=None) -> ConfigResUNet:
    net = ConfigResUNet(channels, in_channels, slope)
    if seed is not None:
        kaiming_reset(net, seed)
    return net
