"""Seeded synthetic workloads of BASELINE.json (configs 0-4).

Shared conventions (BASELINE.json configs[0] "Shared conventions"; SURVEY
§8(d)): cylinder-masked grid in unit-cylinder coordinates; 16 point
electrodes per ring; measurement order of `generate_protocol` on all
electrodes as one ring (M = n(n-3), `pkg/src/d2ip/geometry.py:265-277`);
J[m, v] = s_{m,v} exp(-d(v, m)/0.3), s ~ N(0, 1), d = distance from the voxel
centre to the centroid of the measurement's four electrodes; dv = J sigma_true
+ N(0, (0.01 RMS(J sigma_true))^2); z = 0.1 U[0, 1) with C_z channels.

Choices the BASELINE text leaves open (recorded in DESIGN.md):
  * cfg0 inclusion centre (0.25, -0.2, 0.5);
  * cfg2/cfg4 ring heights 0.2/0.4/0.6/0.8; C_z = 8 for cfg2-4;
  * heart ellipsoid centre (0, 0.35, 0.5), semi-axes (0.15, 0.15, 0.15);
  * frame t = i - 1 for frame i in the sin() waveforms;
  * random streams: J signs default_rng(seed); measurement noise
    default_rng([seed, 1]); cfg3 inclusion scaling default_rng([seed, 3]).
These are inputs, not outputs: the oracle and the GPU path consume the same
arrays, so parity does not depend on them.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field, replace

import numpy as np

from .forward import MaskedSensitivity, VoltageFrame, VoltageSequence
from .geometry import GridGeometry, adjacent_protocol, cylinder_mask, ring_electrodes, vectorize
from .priornet import ResUNetConfig


@dataclass(frozen=True)
class WorkloadSpec:
    name: str
    grid: tuple
    ring_heights: tuple
    channels: tuple
    in_channels: int
    frames: int
    iters_warm: int
    iters_first: int
    iters_next: int
    precision: str = "tf32"     # convolution operand precision: fp32 | tf32 | bf16
    phantom: str = "breathing"  # "ellipsoid" (cfg0) | "breathing" (cfg1-4)
    sequences: int = 1          # cfg3: independent sequences
    joint_frames: int = 0       # cfg4: frames optimised jointly in UPWS
    learning_rate: float = 1e-3
    electrodes_per_ring: int = 16
    decay_length: float = 0.3
    noise_rel: float = 0.01
    size_jitter: float = 0.0    # cfg3: +/-20% inclusion scaling per sequence

    @property
    def n_electrodes(self) -> int:
        return self.electrodes_per_ring * len(self.ring_heights)

    @property
    def n_measurements(self) -> int:
        n = self.n_electrodes
        return n * (n - 3)

    def network(self, seed: int = 0) -> ResUNetConfig:
        return ResUNetConfig(channels=self.channels, in_channels=self.in_channels,
                             negative_slope=0.2, noise_scale=0.1, seed=seed)

    def geometry(self) -> GridGeometry:
        return GridGeometry(*self.grid)


CONFIGS = {
    "cfg0": WorkloadSpec("cfg0", (16, 16, 16), (0.5,), (8, 16), 4, 1, 300, 300, 300,
                         precision="fp32", phantom="ellipsoid"),
    "cfg1": WorkloadSpec("cfg1", (32, 32, 32), (0.3, 0.7), (16, 32, 64), 8, 20, 2000, 100, 100,
                         precision="tf32"),
    "cfg2": WorkloadSpec("cfg2", (64, 64, 32), (0.2, 0.4, 0.6, 0.8), (16, 32, 64, 128), 8, 100,
                         1000, 50, 50, precision="tf32"),
    "cfg3": WorkloadSpec("cfg3", (32, 32, 32), (0.3, 0.7), (16, 32, 64), 8, 50, 2000, 100, 100,
                         precision="tf32", sequences=64, size_jitter=0.2),
    "cfg4": WorkloadSpec("cfg4", (96, 96, 48), (0.2, 0.4, 0.6, 0.8), (32, 64, 128, 256), 8, 100,
                         1000, 50, 50, precision="bf16", joint_frames=16),
}


def voxel_centres(grid: GridGeometry) -> np.ndarray:
    """(Q, 3) xyz in canonical q order."""
    ys, xs, zs = grid.axis_centers()
    R, C, P = grid.shape
    yy = np.broadcast_to(ys[None, :, None], (P, R, C))
    xx = np.broadcast_to(xs[None, None, :], (P, R, C))
    zz = np.broadcast_to(zs[:, None, None], (P, R, C))
    return np.stack([xx.ravel(), yy.ravel(), zz.ravel()], axis=1)


def measurement_centroids(spec: WorkloadSpec) -> np.ndarray:
    pos = ring_electrodes(spec.electrodes_per_ring, spec.ring_heights)
    quads = adjacent_protocol(spec.n_electrodes)
    return pos[quads].mean(axis=1)  # (M, 3)


def jacobian(spec: WorkloadSpec, seed: int = 0, row_chunk: int = 256) -> MaskedSensitivity:
    """Masked fp32 J (M x V), columns in canonical q order of the mask.

    The sign field is drawn sequentially from one default_rng(seed) stream (row chunks
    in order); the distance envelope of each chunk is computed on a thread pool (numpy
    releases the GIL), with the same fp64 operations in the same order as a
    ((dx^2 + dy^2) + dz^2) reduction, so the result does not depend on the pool."""
    from concurrent.futures import ThreadPoolExecutor
    import os

    grid = spec.geometry()
    mask = cylinder_mask(grid)
    cq = voxel_centres(grid)[vectorize(mask)]          # (V, 3)
    cent = measurement_centroids(spec)                  # (M, 3)
    M, V = cent.shape[0], cq.shape[0]
    rng = np.random.default_rng(seed)
    out = np.empty((M, V), dtype=np.float32)
    cx, cy, cz = (np.ascontiguousarray(cq[:, k]) for k in range(3))

    def envelope(r0, r1):
        dx = cx[None, :] - cent[r0:r1, 0:1]
        d2 = dx * dx
        dy = cy[None, :] - cent[r0:r1, 1:2]
        d2 += dy * dy
        dz = cz[None, :] - cent[r0:r1, 2:3]
        d2 += dz * dz
        np.sqrt(d2, out=d2)
        d2 /= -spec.decay_length
        np.exp(d2, out=d2)
        out[r0:r1] *= d2.astype(np.float32)

    chunks = [(r0, min(M, r0 + row_chunk)) for r0 in range(0, M, row_chunk)]
    workers = max(1, min(len(chunks), os.cpu_count() or 1))
    with ThreadPoolExecutor(max_workers=workers) as pool:
        futs = []
        for r0, r1 in chunks:
            out[r0:r1] = rng.standard_normal((r1 - r0, V), dtype=np.float32)
            futs.append(pool.submit(envelope, r0, r1))
        for f in futs:
            f.result()
    return MaskedSensitivity(out, mask, grid.ref_id, f"adjacent{spec.n_electrodes}")


def _jacobian_reference_form(spec: WorkloadSpec, seed: int = 0, row_chunk: int = 256) -> np.ndarray:
    """The direct (single-threaded) statement of `jacobian`, kept for the equality test."""
    grid = spec.geometry()
    mask = cylinder_mask(grid)
    cq = voxel_centres(grid)[vectorize(mask)]
    cent = measurement_centroids(spec)
    M, V = cent.shape[0], cq.shape[0]
    rng = np.random.default_rng(seed)
    out = np.empty((M, V), dtype=np.float32)
    for r0 in range(0, M, row_chunk):
        r1 = min(M, r0 + row_chunk)
        s = rng.standard_normal((r1 - r0, V), dtype=np.float32)
        d = np.sqrt(((cq[None, :, :] - cent[r0:r1, None, :]) ** 2).sum(-1))
        out[r0:r1] = s * np.exp(-d / spec.decay_length).astype(np.float32)
    return out


def jacobian_device(spec: WorkloadSpec, seed: int = 0):
    """The same J model generated directly on the GPU (torch RNG, seeded) for
    the large benchmark configs where host generation of M x V normals would
    dominate the setup. Returns (J [M][V] fp32 cuda, mask). Statistically the
    same inputs as `jacobian`, not bit-identical (different RNG)."""
    import torch

    grid = spec.geometry()
    mask = cylinder_mask(grid)
    cq = torch.from_numpy(voxel_centres(grid)[vectorize(mask)]).cuda().float()
    cent = torch.from_numpy(measurement_centroids(spec)).cuda().float()
    g = torch.Generator(device="cuda").manual_seed(int(seed))
    J = torch.empty((cent.shape[0], cq.shape[0]), dtype=torch.float32, device="cuda")
    for r0 in range(0, J.shape[0], 512):
        r1 = min(J.shape[0], r0 + 512)
        d = torch.cdist(cent[r0:r1], cq)
        J[r0:r1] = torch.randn((r1 - r0, cq.shape[0]), generator=g, device="cuda") * torch.exp(-d / spec.decay_length)
    return J, mask


def device_frame(spec: WorkloadSpec, seed: int = 0, t: int = 0):
    """One frame of the large configs (cfg2 / cfg4) built on the GPU: J from
    `jacobian_device`, dv = J sigma_true(t) + 1 % RMS noise (torch RNG, seeded),
    output_map = (min, max) of sigma_true. Returns (J [M][V] cuda, mask, dv
    [M] cuda fp32, output_map)."""
    import torch

    J, mask = jacobian_device(spec, seed)
    grid = spec.geometry()
    truth = sigma_true(spec, t)
    cols = torch.from_numpy(np.ascontiguousarray(vectorize(truth)[np.flatnonzero(vectorize(mask))])).cuda().float()
    clean = J @ cols
    g = torch.Generator(device="cuda").manual_seed(int(seed) + 7919)
    rms = float(clean.pow(2).mean().sqrt())
    dv = clean + torch.randn(clean.shape, generator=g, device="cuda") * (spec.noise_rel * rms)
    lo, hi = float(truth.min()), float(truth.max())
    if lo == hi:
        lo, hi = lo - 0.5, hi + 0.5
    return J, mask, dv, (lo, hi)


def device_frames(spec: WorkloadSpec, seed: int = 0, T: int = 1):
    """T frames of the large configs on the GPU (cfg4's joint warm-start): J from
    `jacobian_device`, dv_t = J sigma_true(t) + 1 % RMS noise, t = 0..T-1; output_map over
    the T frames. Returns (J [M][V] cuda, mask, dv [T][M] cuda fp32, output_map)."""
    import torch

    J, mask = jacobian_device(spec, seed)
    truths = [sigma_true(spec, t) for t in range(T)]
    cols = torch.from_numpy(np.stack([vectorize(tr)[np.flatnonzero(vectorize(mask))] for tr in truths],
                                     axis=1)).cuda().float()
    clean = (J @ cols).T.contiguous()  # [T][M]
    g = torch.Generator(device="cuda").manual_seed(int(seed) + 7919)
    rms = clean.pow(2).mean(dim=1, keepdim=True).sqrt()
    dv = clean + torch.randn(clean.shape, generator=g, device="cuda") * (spec.noise_rel * rms)
    lo, hi = float(min(t.min() for t in truths)), float(max(t.max() for t in truths))
    if lo == hi:
        lo, hi = lo - 0.5, hi + 0.5
    return J, mask, dv, (lo, hi)


def _ellipsoid(grid: GridGeometry, centre, axes) -> np.ndarray:
    ys, xs, zs = grid.axis_centers()
    u = ((xs[None, :, None] - centre[0]) / axes[0]) ** 2
    v = ((ys[:, None, None] - centre[1]) / axes[1]) ** 2
    w = ((zs[None, None, :] - centre[2]) / axes[2]) ** 2
    return (u + v + w) <= 1.0


def sigma_true(spec: WorkloadSpec, t: int, scale: float = 1.0) -> np.ndarray:
    """(R, C, P) fp64 conductivity change at frame t (0-based)."""
    grid = spec.geometry()
    vol = np.zeros(grid.shape, dtype=np.float64)
    if spec.phantom == "ellipsoid":
        vol[_ellipsoid(grid, (0.25, -0.2, 0.5), (0.3 * scale, 0.2 * scale, 0.25 * scale))] = -0.5
        return vol
    lung_amp = -(0.3 + 0.3 * math.sin(2 * math.pi * t / 10))
    axes = (0.25 * scale, 0.35 * scale, 0.3 * scale)
    for cx in (-0.4, 0.4):
        vol[_ellipsoid(grid, (cx, 0.0, 0.5), axes)] = lung_amp
    heart = _ellipsoid(grid, (0.0, 0.35, 0.5), (0.15 * scale, 0.15 * scale, 0.15 * scale))
    vol[heart] = 0.2 * math.sin(2 * math.pi * t / 3)
    return vol * cylinder_mask(grid)


@dataclass
class Workload:
    spec: WorkloadSpec
    seed: int
    matrix: MaskedSensitivity
    truth: np.ndarray          # (T, R, C, P)
    voltages: VoltageSequence
    output_map: tuple

    @property
    def grid(self) -> GridGeometry:
        return self.spec.geometry()


def make_workload(spec: WorkloadSpec | str, seed: int = 0, frames: int | None = None) -> Workload:
    if isinstance(spec, str):
        spec = CONFIGS[spec]
    T = spec.frames if frames is None else frames
    matrix = jacobian(spec, seed)
    scale = 1.0
    if spec.size_jitter:
        scale = 1.0 + spec.size_jitter * (2 * np.random.default_rng([seed, 3]).random() - 1)
    truth = np.stack([sigma_true(spec, t, scale) for t in range(T)])
    qcols = matrix.columns_q()
    noise_rng = np.random.default_rng([seed, 1])
    frames_out = []
    if matrix.values.size > (1 << 26):
        # large configs (cfg2): all frames in one fp64 GEMM over row blocks of J (no
        # full fp64 copy of a GB-sized J; summation order differs from the per-frame
        # matvec below only in rounding, and nothing at these sizes is golden-pinned)
        X = np.stack([vectorize(truth[i])[qcols] for i in range(T)], axis=1)
        cleans = np.empty((matrix.values.shape[0], T))
        for r0 in range(0, cleans.shape[0], 512):
            cleans[r0:r0 + 512] = matrix.values[r0:r0 + 512].astype(np.float64) @ X
    else:
        J64 = matrix.values.astype(np.float64)
    for i in range(T):
        clean = cleans[:, i] if matrix.values.size > (1 << 26) else J64 @ vectorize(truth[i])[qcols]
        rms = math.sqrt(float(np.mean(clean ** 2))) if np.any(clean) else 0.0
        noisy = clean + noise_rng.normal(0.0, spec.noise_rel * rms, size=clean.size) if rms > 0 else clean
        frames_out.append(VoltageFrame(noisy, i + 1))
    lo, hi = float(truth.min()), float(truth.max())
    if lo == hi:
        lo, hi = lo - 0.5, hi + 0.5
    return Workload(spec, seed, matrix, truth, VoltageSequence(frames_out, seed=seed), (lo, hi))


def run_config_for(spec: WorkloadSpec, output_map, seed: int = 0, **overrides):
    """The RunConfig mapping of SURVEY §7.1 (lr 1e-3, l2sq, lambda_TV = 0)."""
    from .pipeline import RunConfig
    from .regularizers import TVWeights

    kw = dict(
        iters_warm=spec.iters_warm, iters_first=spec.iters_first, iters_next=spec.iters_next,
        learning_rate=spec.learning_rate, optimizer_betas=(0.9, 0.999),
        tv_weights=TVWeights(lambda_tv=0.0), seed=seed, network=spec.network(),
        output_map=tuple(output_map), data_norm="l2sq", warm_frame=1,
        precision=spec.precision,
    )
    kw.update(overrides)
    return RunConfig(**kw)


def small_spec(name="mini", grid=(16, 16, 16), channels=(8, 16, 32), in_channels=8,
               rings=(0.3, 0.7), frames=4, **kw) -> WorkloadSpec:
    """Reduced-size workloads for parity tests (oracle finishes in seconds)."""
    return WorkloadSpec(name, grid, rings, channels, in_channels, frames, 12, 6, 4, **kw)
