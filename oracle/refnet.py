"""The reference backbone FastResUNet3D restated in CPU PyTorch — TEST
INFRASTRUCTURE ONLY.

Follows `pkg/src/d2ip/priornet.py`:
  ChannelLayerNorm  :96-108   (shared with oracle.resunet)
  _conv3            :111-117  depthwise 3^3 (groups=C) + pointwise 1^3, or dense 3^3
  SqueezeExcite     :120-131  mean pool -> 1^3 C->C/4 -> SiLU -> 1^3 -> sigmoid -> scale
  ResConv3d         :134-148  SiLU(norm1(conv1 x)) -> norm2(conv2 .) + skip(x) -> SiLU
  ASPP3d            :151-164  dilated 3^3 branches -> concat -> 1^3 project -> norm -> SiLU
  AttentionGate3d   :167-180  SiLU(key_s2(skip) + query(gate)) -> 1^3 score -> sigmoid
                              -> trilinear x2 -> skip * attn
  FastResUNet3D     :183-232  module registration order = state_dict order
Parameters are loaded by the flat state_dict order, so the module tree below
registers its parameters in exactly the reference's order.
"""

from __future__ import annotations

import torch
import torch.nn.functional as F
from torch import nn

from .resunet import ChannelLayerNorm, kaiming_reset


def _conv3(cin, cout, stride=1, depthwise=True):
    if depthwise:
        return nn.Sequential(nn.Conv3d(cin, cin, 3, stride=stride, padding=1, groups=cin), nn.Conv3d(cin, cout, 1))
    return nn.Conv3d(cin, cout, 3, stride=stride, padding=1)


class SE(nn.Module):
    def __init__(self, c, reduction=4):
        super().__init__()
        hid = max(c // reduction, 1)
        self.fc1 = nn.Conv3d(c, hid, 1)
        self.fc2 = nn.Conv3d(hid, c, 1)

    def forward(self, x):
        g = x.mean(dim=(2, 3, 4), keepdim=True)
        return x * torch.sigmoid(self.fc2(F.silu(self.fc1(g))))


class ResBlock(nn.Module):
    def __init__(self, cin, cout, stride=1, depthwise=True):
        super().__init__()
        self.conv1 = _conv3(cin, cout, stride, depthwise)
        self.norm1 = ChannelLayerNorm(cout)
        self.conv2 = _conv3(cout, cout, 1, depthwise)
        self.norm2 = ChannelLayerNorm(cout)
        self.skip = nn.Conv3d(cin, cout, 1, stride=stride)

    def forward(self, x):
        h = F.silu(self.norm1(self.conv1(x)))
        return F.silu(self.norm2(self.conv2(h)) + self.skip(x))


class ASPP(nn.Module):
    def __init__(self, c, dilations):
        super().__init__()
        self.branches = nn.ModuleList(nn.Conv3d(c, c, 3, padding=d, dilation=d) for d in dilations)
        self.project = nn.Conv3d(c * len(dilations), c, 1)
        self.norm = ChannelLayerNorm(c)

    def forward(self, x):
        return F.silu(self.norm(self.project(torch.cat([b(x) for b in self.branches], 1))))


class AttGate(nn.Module):
    def __init__(self, cs, cg, ci):
        super().__init__()
        self.key = nn.Conv3d(cs, ci, 1, stride=2)
        self.query = nn.Conv3d(cg, ci, 1)
        self.score = nn.Conv3d(ci, 1, 1)

    def forward(self, skip, gate):
        a = torch.sigmoid(self.score(F.silu(self.key(skip) + self.query(gate))))
        return skip * F.interpolate(a, size=skip.shape[2:], mode="trilinear", align_corners=False)


class OracleFastResUNet(nn.Module):
    def __init__(self, base_channels=8, use_depthwise=True, aspp_dilations=(1, 2, 4)):
        super().__init__()
        b = base_channels
        ch = [b, 2 * b, 4 * b, 8 * b]
        self.stem = nn.Sequential(nn.Conv3d(1, b, 3, padding=1), ChannelLayerNorm(b), nn.SiLU())
        self.enc_se = nn.ModuleList(SE(ch[i]) for i in range(3))
        self.enc_block = nn.ModuleList(ResBlock(ch[i], ch[i + 1], 2, use_depthwise) for i in range(3))
        self.bottleneck = ASPP(ch[3], tuple(aspp_dilations))
        self.dec_att = nn.ModuleList(AttGate(ch[i], ch[i + 1], max(ch[i] // 2, 4)) for i in reversed(range(3)))
        self.dec_block = nn.ModuleList(ResBlock(ch[i + 1] + ch[i], ch[i], 1, use_depthwise)
                                       for i in reversed(range(3)))
        self.tail = nn.Conv3d(b, 1, 3, padding=1)

    def forward(self, z):
        squeeze = z.ndim == 3
        x = self.stem(z[None, None] if squeeze else z)
        skips = []
        for se, blk in zip(self.enc_se, self.enc_block):
            s = se(x)
            skips.append(s)
            x = blk(s)
        x = self.bottleneck(x)
        for att, blk, s in zip(self.dec_att, self.dec_block, reversed(skips)):
            g = att(s, x)
            x = F.interpolate(x, size=g.shape[2:], mode="trilinear", align_corners=False)
            x = blk(torch.cat([x, g], 1))
        out = torch.sigmoid(self.tail(x))
        return out[0, 0] if squeeze else out[:, 0]


def build_oracle_refnet(base_channels=8, use_depthwise=True, aspp_dilations=(1, 2, 4), seed=None):
    net = OracleFastResUNet(base_channels, use_depthwise, aspp_dilations)
    if seed is not None:
        kaiming_reset(net, seed)
    return net
