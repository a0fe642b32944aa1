"""Sensitivity-operator assembly on the GPU and the operator / voltage file
formats.

Drop-in names of `pkg/src/d2ip/forward.py`:
  assemble_sensitivity(grid, array, protocol)  forward.py:69-92   (device fp64, returned on the host)
  normalize_sensitivity(matrix)                forward.py:95-112
  save_matrix / load_matrix                    forward.py:221-252 (raw little-endian fp64 + JSON sidecar)
  save_voltages / load_voltages                forward.py:255-289
B200-native additions (the configs where the reference's (M, Q, 3) fp64
arrays do not fit the host):
  assemble_masked_device(grid, array, protocol, mask)  fp32 [M][V] on the GPU, never on the host
  load_matrix_device(path, mask)                       streams row blocks of a saved operator to the GPU
Geometry objects are duck-typed like the reference's: grid.voxel_centers(),
grid.pitch, grid.voxel_volume, grid.ref_id; array.positions_array(),
array.count; protocol.pairs_array(), protocol.count, protocol.ref_id.
"""

from __future__ import annotations

import ctypes as C
import json

import numpy as np

from . import _native as N
from .errors import DegenerateOperatorError, FormatError
from .forward import SensitivityMatrix, VoltageFrame, VoltageSequence
from .geometry import vectorize


def _check_protocol(array, protocol):
    # forward.py:72-76
    if protocol.count == 0:
        raise ValueError("protocol has no measurement pairs")
    if np.asarray(protocol.pairs_array()).max() >= array.count:
        raise ValueError("protocol references electrodes beyond the array")


def _device_assemble(grid, array, protocol, normalize, q_of_col=None):
    import torch

    from .engine import require_cuda

    require_cuda()
    _check_protocol(array, protocol)
    dev = "cuda"
    centers = torch.from_numpy(np.ascontiguousarray(grid.voxel_centers(), dtype=np.float64)).to(dev)
    elec = torch.from_numpy(np.ascontiguousarray(array.positions_array(), dtype=np.float64)).to(dev)
    quads = torch.from_numpy(np.ascontiguousarray(protocol.pairs_array(), dtype=np.int32)).to(dev)
    Q, E, M = centers.shape[0], elec.shape[0], quads.shape[0]
    out = torch.empty((M, Q), dtype=torch.float64, device=dev)
    norms = torch.empty(M, dtype=torch.float64, device=dev)
    Jm, V, Vp, qc = None, 0, 0, None
    if q_of_col is not None:
        V = int(q_of_col.size)
        Vp = (V + 3) // 4 * 4
        Jm = torch.empty((M, Vp), dtype=torch.float32, device=dev)
        qc = torch.from_numpy(np.ascontiguousarray(q_of_col, dtype=np.int32)).to(dev)
    min_dist = min(grid.pitch) / 2  # forward.py:62
    st = C.c_void_p(torch.cuda.current_stream().cuda_stream)
    N.check(N.lib().d2ip_assemble_sensitivity(
        C.c_void_p(centers.data_ptr()), Q, C.c_void_p(elec.data_ptr()), E, C.c_void_p(quads.data_ptr()), M,
        float(min_dist), float(grid.voxel_volume), 1 if normalize else 0, C.c_void_p(out.data_ptr()),
        C.c_void_p(norms.data_ptr()), C.c_void_p(Jm.data_ptr()) if Jm is not None else None, V, Vp,
        C.c_void_p(qc.data_ptr()) if qc is not None else None, st), "assemble_sensitivity")
    return out, norms, Jm


def assemble_sensitivity(grid, array, protocol) -> SensitivityMatrix:
    """`forward.py:69-92` computed on the GPU in fp64 (unnormalised)."""
    out, _, _ = _device_assemble(grid, array, protocol, normalize=False)
    return SensitivityMatrix(out.cpu().numpy(), False, False, grid.ref_id, protocol.ref_id)


def normalize_sensitivity(matrix: SensitivityMatrix) -> SensitivityMatrix:
    """`forward.py:95-112`: unit Euclidean rows; identically-zero rows raise."""
    norms = np.linalg.norm(matrix.values, axis=1)
    zero_rows = np.flatnonzero(norms == 0)
    if zero_rows.size:
        raise DegenerateOperatorError(f"sensitivity rows {zero_rows.tolist()} are identically zero")
    return SensitivityMatrix(matrix.values / norms[:, None], True, True, matrix.grid_ref, matrix.protocol_ref)


def assemble_masked_device(grid, array, protocol, mask, normalize: bool = True):
    """Normalised operator restricted to `mask`, fp32 [M][V] on the GPU with the
    columns in canonical q order (what `DeviceNet.set_J_device` takes). The fp64
    operator lives only on the device. Returns (J, norms fp64)."""
    q_of_col = np.flatnonzero(vectorize(np.asarray(mask, dtype=bool)))
    out, norms, Jm = _device_assemble(grid, array, protocol, normalize, q_of_col)
    if normalize and bool((norms == 0).any()):
        zero = np.flatnonzero((norms == 0).cpu().numpy())
        raise DegenerateOperatorError(f"sensitivity rows {zero.tolist()} are identically zero")
    del out
    return Jm[:, : q_of_col.size].contiguous(), norms


# ---------------------------------------------------------------------------
# Persistence: raw little-endian float64 payload plus a JSON sidecar
# (forward.py:197-289; the same bytes and keys, so files interoperate).


def _sidecar_path(path) -> str:
    return f"{path}.json"


def _write_payload(path, array: np.ndarray) -> None:
    with open(path, "wb") as fh:
        fh.write(np.ascontiguousarray(array, dtype="<f8").tobytes())


def _read_payload(path, count: int) -> np.ndarray:
    with open(path, "rb") as fh:
        raw = fh.read()
    if len(raw) != count * 8:
        raise FormatError(f"{path}: expected {count * 8} payload bytes per sidecar, found {len(raw)}")
    return np.frombuffer(raw, dtype="<f8").astype(np.float64)


def save_matrix(matrix: SensitivityMatrix, path) -> None:
    _write_payload(path, matrix.values)
    doc = {"M": matrix.n_measurements, "Q": matrix.n_voxels, "normalized": matrix.normalized,
           "projected": matrix.projected, "grid_ref": matrix.grid_ref, "protocol_ref": matrix.protocol_ref}
    with open(_sidecar_path(path), "w") as fh:
        json.dump(doc, fh, sort_keys=True, indent=1)


def _matrix_doc(path):
    with open(_sidecar_path(path)) as fh:
        doc = json.load(fh)
    try:
        return doc, int(doc["M"]), int(doc["Q"])
    except KeyError as exc:
        raise FormatError(f"malformed matrix sidecar for {path}: missing {exc}") from exc


def load_matrix(path) -> SensitivityMatrix:
    doc, m, q = _matrix_doc(path)
    try:
        values = _read_payload(path, m * q).reshape(m, q)
        return SensitivityMatrix(values, bool(doc["normalized"]), bool(doc["projected"]), doc["grid_ref"],
                                 doc["protocol_ref"])
    except KeyError as exc:
        raise FormatError(f"malformed matrix sidecar for {path}: missing {exc}") from exc


def load_matrix_device(path, mask, rows_per_block: int = 256):
    """A saved operator's masked fp32 block on the GPU, [M][V] in canonical
    column order, streamed in row blocks (the host holds one block at a time,
    never the fp64 M x Q array)."""
    import torch

    doc, m, q = _matrix_doc(path)
    import os

    if os.path.getsize(path) != m * q * 8:
        raise FormatError(f"{path}: expected {m * q * 8} payload bytes per sidecar, found {os.path.getsize(path)}")
    cols = torch.from_numpy(np.flatnonzero(vectorize(np.asarray(mask, dtype=bool)))).cuda()
    if int(np.asarray(mask).size) != q:
        raise ValueError(f"mask has {int(np.asarray(mask).size)} voxels, operator has {q}")
    J = torch.empty((m, cols.numel()), dtype=torch.float32, device="cuda")
    raw = np.memmap(path, dtype="<f8", mode="r", shape=(m, q))
    for r0 in range(0, m, rows_per_block):
        r1 = min(m, r0 + rows_per_block)
        blk = torch.from_numpy(np.ascontiguousarray(raw[r0:r1])).cuda()
        J[r0:r1] = blk.index_select(1, cols).float()
    del raw
    return J, doc


def save_voltages(seq: VoltageSequence, path) -> None:
    _write_payload(path, np.stack([f.values for f in seq.frames], axis=0))
    doc = {"M": seq.n_measurements, "T": seq.n_frames, "reference_mode": seq.reference_mode,
           "snr_db": seq.snr_db, "seed": seq.seed, "protocol_ref": seq.protocol_ref}
    with open(_sidecar_path(path), "w") as fh:
        json.dump(doc, fh, sort_keys=True, indent=1)


def load_voltages(path) -> VoltageSequence:
    with open(_sidecar_path(path)) as fh:
        doc = json.load(fh)
    try:
        m, t = int(doc["M"]), int(doc["T"])
        flat = _read_payload(path, m * t).reshape(t, m)
        frames = [VoltageFrame(flat[i], i + 1, snr_db=doc["snr_db"]) for i in range(t)]
        return VoltageSequence(frames=frames, reference_mode=doc["reference_mode"], snr_db=doc["snr_db"],
                               seed=doc["seed"], protocol_ref=doc.get("protocol_ref"))
    except KeyError as exc:
        raise FormatError(f"malformed voltage sidecar for {path}: missing {exc}") from exc
