"""Lead-field sensitivity operator restated in NumPy -- TEST INFRASTRUCTURE ONLY.

Follows `pkg/src/d2ip/forward.py`:
  _lead_fields          :58-66   f_e(q) = -(c_q - p_e) / (4 pi max(|c_q - p_e|, min_pitch/2)^3)
  assemble_sensitivity  :69-92   S[m][q] = -(f_d+ - f_d-).(f_m+ - f_m-) * voxel_volume
  normalize_sensitivity :95-112  unit Euclidean rows
on plain arrays (voxel centres, electrode positions, quadruples), so the GPU
kernel (csrc/sensitivity.cu) can be checked without the reference installed.
Pinned against tests/golden/sensitivity.npz (written by the real reference).
"""

import math

import numpy as np


def oracle_lead_fields(centers, positions, min_dist):
    diff = centers[None, :, :] - positions[:, None, :]
    dist = np.maximum(np.linalg.norm(diff, axis=2), min_dist)
    return -diff / (4 * math.pi * dist**3)[:, :, None]


def oracle_assemble(centers, positions, quads, min_dist, voxel_volume):
    fields = oracle_lead_fields(np.asarray(centers, np.float64), np.asarray(positions, np.float64), min_dist)
    quads = np.asarray(quads)
    gd = fields[quads[:, 0]] - fields[quads[:, 1]]
    gm = fields[quads[:, 2]] - fields[quads[:, 3]]
    return -np.einsum("mqk,mqk->mq", gd, gm) * voxel_volume


def oracle_normalize(values):
    norms = np.linalg.norm(values, axis=1)
    return values / norms[:, None], norms
