"""Golden fixtures of the reference's sensitivity operator and file formats,
from the REAL reference package (`pkg/src/d2ip/forward.py`, `geometry.py`).

Run in the build container only:  python tests/golden/make_golden_sensitivity.py
Writes tests/golden/sensitivity.npz: the geometry arrays the GPU path needs
(voxel centres, electrode positions, quadruples, pitch, voxel volume, refs),
the unnormalised operator and its row norms (assemble_sensitivity +
normalize_sensitivity, forward.py:58-112) for a 6x6x4 thorax-box grid with
the default 2 x 16 belt, plus the exact bytes save_matrix / save_voltages
write (forward.py:197-289) so format parity is checked byte for byte.
"""

import json
import sys
import tempfile
from pathlib import Path

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")

from d2ip import forward as F  # noqa: E402
from d2ip import geometry as G  # noqa: E402

OUT = Path(__file__).resolve().parent


def main():
    grid = G.build_grid(6, 6, 4, G.THORAX_BOX)
    array = G.default_electrode_array(grid)
    proto = G.generate_protocol(array)
    raw = F.assemble_sensitivity(grid, array, proto)
    norm = F.normalize_sensitivity(raw)
    rng = np.random.default_rng(3)
    frames = [F.VoltageFrame(rng.normal(size=raw.n_measurements), i + 1) for i in range(3)]
    seq = F.VoltageSequence(frames, seed=3, protocol_ref=proto.ref_id)
    with tempfile.TemporaryDirectory() as d:
        F.save_matrix(norm, f"{d}/J.bin")
        F.save_voltages(seq, f"{d}/dv.bin")
        jbytes = Path(f"{d}/J.bin").read_bytes()
        jside = Path(f"{d}/J.bin.json").read_text()
        vbytes = Path(f"{d}/dv.bin").read_bytes()
        vside = Path(f"{d}/dv.bin.json").read_text()
    np.savez_compressed(
        OUT / "sensitivity.npz",
        centers=grid.voxel_centers(), positions=array.positions_array(), quads=proto.pairs_array(),
        pitch=np.array(grid.pitch), voxel_volume=np.array(grid.voxel_volume), shape=np.array(grid.shape),
        grid_ref=np.array(grid.ref_id), protocol_ref=np.array(proto.ref_id),
        raw=raw.values, norms=np.linalg.norm(raw.values, axis=1), normalized=norm.values,
        dv=np.stack([f.values for f in frames]),
        J_bin=np.frombuffer(jbytes, dtype=np.uint8), J_side=np.array(jside),
        dv_bin=np.frombuffer(vbytes, dtype=np.uint8), dv_side=np.array(vside))
    print("M", raw.n_measurements, "Q", raw.n_voxels, "ref", grid.ref_id, proto.ref_id)


if __name__ == "__main__":
    main()
