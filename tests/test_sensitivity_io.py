"""Sensitivity assembly and operator / voltage file formats
(§8(f) #4) against the REAL reference (tests/golden/sensitivity.npz, written by
tests/golden/make_golden_sensitivity.py from pkg/src/d2ip/forward.py)."""

import json

import numpy as np
import pytest
import torch

from conftest import GOLDEN
from oracle.sensitivity import oracle_assemble, oracle_normalize
from paper_2507_14046_b200 import DegenerateOperatorError, FormatError, SensitivityMatrix
from paper_2507_14046_b200 import sensitivity as S
from paper_2507_14046_b200.geometry import vectorize


@pytest.fixture(scope="module")
def gold():
    return np.load(GOLDEN / "sensitivity.npz")


class _Grid:
    def __init__(self, g):
        self._c, self.pitch, self.voxel_volume = g["centers"], tuple(g["pitch"]), float(g["voxel_volume"])
        self.shape, self.ref_id = tuple(int(v) for v in g["shape"]), str(g["grid_ref"])

    def voxel_centers(self):
        return self._c


class _Array:
    def __init__(self, g):
        self._p = g["positions"]
        self.count = self._p.shape[0]

    def positions_array(self):
        return self._p


class _Proto:
    def __init__(self, quads, ref=""):
        self._q, self.count, self.ref_id = np.asarray(quads), len(quads), ref

    def pairs_array(self):
        return self._q


def test_oracle_matches_reference_bitwise(gold):
    raw = oracle_assemble(gold["centers"], gold["positions"], gold["quads"], min(gold["pitch"]) / 2,
                          float(gold["voxel_volume"]))
    np.testing.assert_array_equal(raw, gold["raw"])
    np.testing.assert_array_equal(oracle_normalize(raw)[0], gold["normalized"])


def test_normalize_matches_reference_bitwise(gold):
    m = S.normalize_sensitivity(SensitivityMatrix(gold["raw"], False, False, "g", "p"))
    np.testing.assert_array_equal(m.values, gold["normalized"])
    assert m.normalized and m.projected
    zero = gold["raw"].copy()
    zero[3] = 0.0
    with pytest.raises(DegenerateOperatorError):
        S.normalize_sensitivity(SensitivityMatrix(zero, False, False, "g", "p"))


def test_protocol_validation(gold):
    with pytest.raises(ValueError):
        S._check_protocol(_Array(gold), _Proto(np.zeros((0, 4), int)))
    bad = gold["quads"].copy()
    bad[0, 0] = 99
    with pytest.raises(ValueError):
        S._check_protocol(_Array(gold), _Proto(bad))


def test_file_formats_byte_identical(gold, tmp_path):
    from paper_2507_14046_b200 import VoltageFrame, VoltageSequence
    m = SensitivityMatrix(gold["normalized"], True, True, str(gold["grid_ref"]), str(gold["protocol_ref"]))
    S.save_matrix(m, tmp_path / "J.bin")
    assert (tmp_path / "J.bin").read_bytes() == gold["J_bin"].tobytes()
    assert json.loads((tmp_path / "J.bin.json").read_text()) == json.loads(str(gold["J_side"]))
    assert (tmp_path / "J.bin.json").read_text() == str(gold["J_side"])
    seq = VoltageSequence([VoltageFrame(v, i + 1) for i, v in enumerate(gold["dv"])], seed=3,
                          protocol_ref=str(gold["protocol_ref"]))
    S.save_voltages(seq, tmp_path / "dv.bin")
    assert (tmp_path / "dv.bin").read_bytes() == gold["dv_bin"].tobytes()
    assert (tmp_path / "dv.bin.json").read_text() == str(gold["dv_side"])
    back = S.load_matrix(tmp_path / "J.bin")
    np.testing.assert_array_equal(back.values, gold["normalized"])
    assert back.grid_ref == str(gold["grid_ref"]) and back.normalized
    vs = S.load_voltages(tmp_path / "dv.bin")
    np.testing.assert_array_equal(vs.as_matrix().T, gold["dv"])
    assert vs.seed == 3 and vs.n_frames == 3


def test_file_format_errors(gold, tmp_path):
    (tmp_path / "J.bin").write_bytes(gold["J_bin"].tobytes()[:-8])
    (tmp_path / "J.bin.json").write_text(str(gold["J_side"]))
    with pytest.raises(FormatError):
        S.load_matrix(tmp_path / "J.bin")
    doc = json.loads(str(gold["J_side"]))
    del doc["Q"]
    (tmp_path / "K.bin").write_bytes(gold["J_bin"].tobytes())
    (tmp_path / "K.bin.json").write_text(json.dumps(doc))
    with pytest.raises(FormatError):
        S.load_matrix(tmp_path / "K.bin")


@pytest.mark.gpu
def test_device_assembly_matches_reference(gold):
    grid, arr, proto = _Grid(gold), _Array(gold), _Proto(gold["quads"], str(gold["protocol_ref"]))
    m = S.assemble_sensitivity(grid, arr, proto)
    ref = gold["raw"]
    assert m.values.shape == ref.shape and not m.normalized
    # fp64 on both sides; only last-bit differences (division / sqrt implementations)
    assert np.abs(m.values - ref).max() <= 1e-13 * np.abs(ref).max()
    n = S.normalize_sensitivity(m)
    assert np.abs(n.values - gold["normalized"]).max() <= 1e-13


@pytest.mark.gpu
def test_device_masked_block_matches_reference(gold):
    grid, arr, proto = _Grid(gold), _Array(gold), _Proto(gold["quads"], str(gold["protocol_ref"]))
    shape = grid.shape
    mask = np.zeros(shape, dtype=bool)
    mask[1:5, 1:5, :] = True
    J, norms = S.assemble_masked_device(grid, arr, proto, mask)
    cols = np.flatnonzero(vectorize(mask))
    want = gold["normalized"][:, cols].astype(np.float32)
    np.testing.assert_allclose(J.cpu().numpy(), want, rtol=1e-6, atol=1e-7)
    np.testing.assert_allclose(norms.cpu().numpy(), gold["norms"], rtol=1e-13)


@pytest.mark.gpu
def test_load_matrix_device(gold, tmp_path):
    m = SensitivityMatrix(gold["normalized"], True, True, str(gold["grid_ref"]), str(gold["protocol_ref"]))
    S.save_matrix(m, tmp_path / "J.bin")
    shape = tuple(int(v) for v in gold["shape"])
    mask = np.ones(shape, dtype=bool)
    mask[0] = False
    J, doc = S.load_matrix_device(tmp_path / "J.bin", mask, rows_per_block=100)
    cols = np.flatnonzero(vectorize(mask))
    np.testing.assert_array_equal(J.cpu().numpy(), gold["normalized"][:, cols].astype(np.float32))
    assert doc["normalized"] is True
