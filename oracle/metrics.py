"""Parity judges — TEST INFRASTRUCTURE ONLY.

`mssim` restates the reference's slice-wise SSIM (`pkg/src/d2ip/metrics.py:72-100`:
11x11 Gaussian window sigma 1.5, K1 0.01 / K2 0.03, joint dynamic range);
`misfit` is the relative data misfit ||J sigma - dv|| / ||dv|| the north star's
"within 2%" criterion is stated on.
"""

from __future__ import annotations

import numpy as np
from scipy.ndimage import gaussian_filter

_SIGMA = 1.5
_TRUNC = 5.0 / _SIGMA


def _ssim_slice(a, b, drange):
    smooth = lambda im: gaussian_filter(im, _SIGMA, truncate=_TRUNC)  # noqa: E731
    mu_a, mu_b = smooth(a), smooth(b)
    var_a = smooth(a * a) - mu_a ** 2
    var_b = smooth(b * b) - mu_b ** 2
    cov = smooth(a * b) - mu_a * mu_b
    c1 = (0.01 * drange) ** 2
    c2 = (0.03 * drange) ** 2
    num = (2 * mu_a * mu_b + c1) * (2 * cov + c2)
    den = (mu_a ** 2 + mu_b ** 2 + c1) * (var_a + var_b + c2)
    return float(np.mean(num / den))


def mssim(x, ref) -> float:
    a = np.asarray(x, dtype=np.float64)
    b = np.asarray(ref, dtype=np.float64)
    if a.shape != b.shape or a.ndim != 3:
        raise ValueError(f"expected equal 3D shapes, got {a.shape} vs {b.shape}")
    lo, hi = min(a.min(), b.min()), max(a.max(), b.max())
    if hi == lo:
        return 1.0
    return float(np.mean([_ssim_slice(a[:, :, p], b[:, :, p], hi - lo) for p in range(a.shape[2])]))


def misfit(J, qcols, volume, dv) -> float:
    """||J vec(volume)[mask] - dv|| / ||dv|| in float64."""
    q = np.transpose(np.asarray(volume, np.float64), (2, 0, 1)).reshape(-1)[qcols]
    r = np.asarray(J, np.float64) @ q - np.asarray(dv, np.float64)
    return float(np.linalg.norm(r) / np.linalg.norm(dv))
