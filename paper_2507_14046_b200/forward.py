"""Operator and measurement containers of the drop-in surface.

``SensitivityMatrix`` mirrors the reference's dense, read-only fp64 M x Q
operator (`pkg/src/d2ip/forward.py:30-55`); inside the reference loop it is
cast to a dense fp32 tensor (`pkg/src/d2ip/pipeline.py:273`) and used as
``operator @ vec(mapped)`` (`pipeline.py:279`).

``MaskedSensitivity`` is the B200-native form the BASELINE configs define: the
M x V block of J over the voxels of a mask (V << Q), stored fp32. A dense
operator whose columns are zero outside the mask is arithmetically the same
operator; `as_masked` converts either form, and the device runner uploads the
masked block once per runner, column-permuted into the network's memory order.

``VoltageFrame`` / ``VoltageSequence`` mirror `forward.py:125-174`.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .geometry import vectorize

REFERENCE_MODES = ("empty_background", "first_frame")


@dataclass(frozen=True)
class SensitivityMatrix:
    """Dense M x Q linear operator (reference layout, fp64, read-only)."""

    values: np.ndarray
    normalized: bool = True
    projected: bool = True
    grid_ref: str = ""
    protocol_ref: str = ""

    def __post_init__(self):
        vals = np.ascontiguousarray(self.values, dtype=np.float64)
        if vals.ndim != 2:
            raise ValueError(f"sensitivity matrix must be 2D, got shape {vals.shape}")
        if not np.all(np.isfinite(vals)):
            raise ValueError("sensitivity matrix contains non-finite entries")
        vals.setflags(write=False)
        object.__setattr__(self, "values", vals)

    @property
    def n_measurements(self) -> int:
        return self.values.shape[0]

    @property
    def n_voxels(self) -> int:
        return self.values.shape[1]


@dataclass(frozen=True)
class MaskedSensitivity:
    """M x V operator over the masked voxels, columns in canonical order q.

    ``mask`` is the (R, C, P) bool volume; column j of ``values`` belongs to the
    j-th True entry of ``vectorize(mask)`` (q = ((p*R)+r)*C+c ordering).
    ``n_voxels`` reports the full-grid Q so driver validation matches the
    reference (`pkg/src/d2ip/pipeline.py:457-458`).
    """

    values: np.ndarray
    mask: np.ndarray
    grid_ref: str = ""
    protocol_ref: str = ""

    def __post_init__(self):
        vals = np.asarray(self.values)
        if vals.dtype not in (np.float32, np.float64):
            vals = vals.astype(np.float32)
        vals = np.ascontiguousarray(vals)
        mask = np.ascontiguousarray(np.asarray(self.mask, dtype=bool))
        if vals.ndim != 2:
            raise ValueError(f"sensitivity block must be 2D, got shape {vals.shape}")
        if mask.ndim != 3:
            raise ValueError(f"mask must be an (R, C, P) volume, got shape {mask.shape}")
        if int(mask.sum()) != vals.shape[1]:
            raise ValueError(
                f"mask selects {int(mask.sum())} voxels but the block has {vals.shape[1]} columns"
            )
        vals.setflags(write=False)
        mask.setflags(write=False)
        object.__setattr__(self, "values", vals)
        object.__setattr__(self, "mask", mask)

    @property
    def n_measurements(self) -> int:
        return self.values.shape[0]

    @property
    def n_voxels(self) -> int:
        return int(self.mask.size)

    @property
    def n_masked(self) -> int:
        return self.values.shape[1]

    def columns_q(self) -> np.ndarray:
        """Canonical index q of every column."""
        return np.flatnonzero(vectorize(self.mask))

    def dense(self) -> SensitivityMatrix:
        """The equal dense M x Q operator (zero columns outside the mask)."""
        full = np.zeros((self.n_measurements, self.n_voxels), dtype=np.float64)
        full[:, self.columns_q()] = self.values
        return SensitivityMatrix(full, True, True, self.grid_ref, self.protocol_ref)


def as_masked(matrix, grid_shape) -> MaskedSensitivity:
    """Masked view of either operator form. A dense operator keeps every
    column (mask = all voxels), exactly the reference's arithmetic."""
    if isinstance(matrix, MaskedSensitivity):
        return matrix
    values = np.asarray(matrix.values)
    if values.shape[1] != int(np.prod(grid_shape)):
        raise ValueError("operator voxel count does not match the grid")
    return MaskedSensitivity(values, np.ones(grid_shape, dtype=bool),
                             getattr(matrix, "grid_ref", ""), getattr(matrix, "protocol_ref", ""))


@dataclass(frozen=True)
class VoltageFrame:
    """One frame of differential boundary measurements (`forward.py:125-139`)."""

    values: np.ndarray
    frame_index: int
    snr_db: float | None = None

    def __post_init__(self):
        vals = np.ascontiguousarray(self.values, dtype=np.float64)
        if vals.ndim != 1:
            raise ValueError(f"voltage frame must be 1D, got shape {vals.shape}")
        if not np.all(np.isfinite(vals)):
            raise ValueError("voltage frame contains non-finite entries")
        object.__setattr__(self, "values", vals)


@dataclass
class VoltageSequence:
    """Ordered voltage frames sharing one protocol (`forward.py:142-174`)."""

    frames: list
    reference_mode: str = "empty_background"
    snr_db: float | None = None
    seed: int | None = None
    protocol_ref: str | None = None

    def __post_init__(self):
        if not self.frames:
            raise ValueError("voltage sequence must hold at least one frame")
        if self.reference_mode not in REFERENCE_MODES:
            raise ValueError(f"unknown reference mode {self.reference_mode!r}")
        m = self.frames[0].values.size
        for i, fr in enumerate(self.frames, start=1):
            if fr.values.size != m:
                raise ValueError("voltage frames have inconsistent lengths")
            if fr.frame_index != i:
                raise ValueError("frame indices must run 1..T contiguously")

    @property
    def n_frames(self) -> int:
        return len(self.frames)

    @property
    def n_measurements(self) -> int:
        return self.frames[0].values.size

    def as_matrix(self) -> np.ndarray:
        return np.stack([f.values for f in self.frames], axis=1)


@dataclass
class ConductivitySequence:
    """Q x T per-frame conductivity changes in canonical voxel order
    (`pkg/src/d2ip/phantom.py:240-272`)."""

    values: np.ndarray
    grid_ref: str
    is_ground_truth: bool
    reference_mode: str
    case: str | None = None
    conductivities: dict | None = None
    method: str | None = None

    def __post_init__(self):
        vals = np.ascontiguousarray(self.values, dtype=np.float64)
        if vals.ndim != 2:
            raise ValueError(f"sequence values must be (Q, T), got shape {vals.shape}")
        if not np.all(np.isfinite(vals)):
            raise ValueError("sequence contains non-finite entries")
        self.values = vals

    @property
    def n_voxels(self) -> int:
        return self.values.shape[0]

    @property
    def n_frames(self) -> int:
        return self.values.shape[1]

    def frame(self, i: int) -> np.ndarray:
        return self.values[:, i - 1]


def forward_project(matrix, dsigma) -> np.ndarray:
    """Measurement-space projection of a conductivity-change vector
    (`pkg/src/d2ip/forward.py:115-122`): ``matrix.values @ vec`` in float64, computed
    on the GPU by the deterministic fp64 kernel `d2ip_project_f64`. Accepts the
    reference's dense operator (Q columns) or the masked block (its masked columns
    of the Q-vector)."""
    import torch

    from . import _native as N
    from .engine import _stream_ptr, require_cuda

    vec = np.asarray(dsigma, dtype=np.float64)
    if vec.shape != (matrix.n_voxels,):
        raise ValueError(f"conductivity vector shape {vec.shape} does not match Q={matrix.n_voxels}")
    if isinstance(matrix, MaskedSensitivity):
        vec = vec[matrix.columns_q()]
    require_cuda()
    A = torch.as_tensor(np.asarray(matrix.values), device="cuda").to(torch.float64).contiguous()
    x = torch.as_tensor(vec, device="cuda").contiguous()
    M, n = A.shape
    y = torch.empty(M, dtype=torch.float64, device="cuda")
    N.check(N.lib().d2ip_project_f64(N.C.c_void_p(A.data_ptr()), n, N.C.c_void_p(x.data_ptr()), M, n,
                                     N.C.c_void_p(y.data_ptr()), N.C.c_void_p(_stream_ptr())), "project_f64")
    return y.cpu().numpy()
