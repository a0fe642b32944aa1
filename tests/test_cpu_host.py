"""Host-side logic on the CPU: API mirror, schema, layouts, workloads, and the
C-ABI library's symbol table (no compute calls without a GPU)."""

import ctypes
import re
from dataclasses import replace
from pathlib import Path

import numpy as np
import pytest
import torch

from conftest import ROOT
from oracle import build_oracle_net
from paper_2507_14046_b200 import (
    NativeLibraryError,
    RunConfig,
    TVWeights,
    ablation_mode,
    count_parameters,
)
from paper_2507_14046_b200 import _native
from paper_2507_14046_b200 import workloads as W
from paper_2507_14046_b200.engine import ColumnMap
from paper_2507_14046_b200.geometry import GridGeometry, adjacent_protocol, cylinder_mask, devectorize, vectorize
from paper_2507_14046_b200.pipeline import (
    LossTrace,
    TraceRecord,
    read_timing_csv,
    read_traces_csv,
    write_timing_csv,
    write_traces_csv,
)
from paper_2507_14046_b200.priornet import (
    ParameterState,
    ResUNetConfig,
    init_parameters,
    kaiming_flat,
    load_checkpoint,
    param_schema,
    save_checkpoint,
)


def header_symbols():
    text = (ROOT / "include" / "d2ip_b200.h").read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(d2ip_\w+)\s*\(", text)))


def test_library_exports_every_header_symbol():
    lib = ctypes.CDLL(str(_native.LIB_PATH))
    syms = header_symbols()
    assert len(syms) >= 25
    for s in syms:
        assert hasattr(lib, s), s
    assert set(syms) == set(_native.exported_symbols())
    assert _native.lib().d2ip_abi_version() == _native.ABI_VERSION


@pytest.mark.skipif(torch.cuda.is_available(), reason="CPU-only check")
def test_gpu_path_fails_loudly_without_cuda():
    from paper_2507_14046_b200.engine import DeviceNet
    spec = W.small_spec()
    with pytest.raises(NativeLibraryError):
        DeviceNet(spec.network(), (16, 16, 16), 10, np.ones((16, 16, 16), bool))


@pytest.mark.parametrize("name,count", [("cfg0", 33065), ("cfg1", 582673), ("cfg2", 2386705), ("cfg4", 9532449)])
def test_param_counts_match_survey(name, count):
    assert count_parameters(W.CONFIGS[name].network()) == count


@pytest.mark.parametrize("channels,cz", [((8, 16), 4), ((16, 32, 64), 8), ((4, 8, 12, 16), 2)])
def test_schema_and_init_match_module_tree(channels, cz):
    cfg = ResUNetConfig(channels=channels, in_channels=cz, seed=3)
    net = build_oracle_net(channels, cz, seed=3)
    sd = net.state_dict()
    schema = param_schema(cfg)
    assert [e.name for e in schema] == list(sd)
    assert [tuple(e.shape) for e in schema] == [tuple(v.shape) for v in sd.values()]
    np.testing.assert_array_equal(kaiming_flat(cfg).numpy(), torch.cat([v.reshape(-1) for v in sd.values()]).numpy())


def test_parameter_state_roundtrip_and_checkpoint(tmp_path):
    cfg = ResUNetConfig(channels=(8, 16), in_channels=4, seed=1)
    st = init_parameters(cfg)
    flat = st.flat(param_schema(cfg))
    assert flat.numel() == count_parameters(cfg)
    c2 = st.clone(provenance="tpp")
    assert c2.checksum() == st.checksum() and c2.provenance == "tpp"
    p = tmp_path / "ck.pt"
    save_checkpoint(p, st, cfg)
    assert load_checkpoint(p, cfg).checksum() == st.checksum()
    from paper_2507_14046_b200 import FormatError
    with pytest.raises(FormatError):
        load_checkpoint(p, ResUNetConfig(channels=(8, 24), in_channels=4))


def test_runconfig_json_roundtrip_and_validation():
    cfg = RunConfig(iters_warm=12, iters_first=6, iters_next=4, network=ResUNetConfig(channels=(8, 16)),
                    disable_tpp=True, output_map=(-0.2, 0.0), precision="tf32")
    doc = cfg.to_json()
    assert doc["stage_ratio"] == "12:6:4"
    assert RunConfig.from_json(doc) == cfg
    d = RunConfig()
    assert d.stage_ratio() == "1800:450:250" and d.learning_rate == 5e-4
    assert d.tv_weights == TVWeights(0.002, 1.0, 0.1, 1e-8)
    assert RunConfig.from_json(d.to_json()) == d
    for bad in (dict(iters_warm=-1), dict(data_norm="huber"), dict(output_map=(0.5, 0.5)), dict(precision="fp8")):
        with pytest.raises(ValueError):
            RunConfig(**bad)
    assert ablation_mode(cfg, {"upws"}).disable_upws
    with pytest.raises(ValueError):
        ablation_mode(cfg, {"warm"})


def test_vectorize_order_and_column_map():
    g = GridGeometry(4, 6, 2)
    vol = np.arange(48).reshape(4, 6, 2)
    v = vectorize(vol)
    r, c, p = 3, 5, 1
    assert v[((p * 4) + r) * 6 + c] == vol[r, c, p]
    np.testing.assert_array_equal(devectorize(v, g.shape), vol)
    mask = np.random.default_rng(0).random((4, 6, 2)) > 0.4
    cm = ColumnMap.from_mask(mask)
    q = np.flatnonzero(vectorize(mask))
    # device column j holds canonical column perm[j], at memory offset vox_of_col[j]
    mem = vol.reshape(-1)  # memory order (r, c, p) == arange
    np.testing.assert_array_equal(mem[cm.vox_of_col], vectorize(vol)[q[cm.perm]])
    assert np.all(np.diff(cm.vox_of_col) > 0)
    assert (cm.col_of_vox >= 0).sum() == mask.sum()


@pytest.mark.parametrize("name,V,M", [("cfg0", 3328, 208), ("cfg1", 25984, 928), ("cfg2", 103296, 3904)])
def test_workload_shapes(name, V, M):
    spec = W.CONFIGS[name]
    assert int(cylinder_mask(spec.geometry()).sum()) == V
    assert spec.n_measurements == M
    assert adjacent_protocol(spec.n_electrodes).shape == (M, 4)


def test_workload_cfg0_generation():
    wl = W.make_workload("cfg0", seed=0)
    assert wl.matrix.values.shape == (208, 3328) and wl.matrix.values.dtype == np.float32
    assert wl.voltages.n_frames == 1
    lo, hi = wl.output_map
    assert lo == -0.5 and hi == 0.0


def test_trace_and_timing_csv(tmp_path):
    tr = LossTrace()
    for k, d in enumerate([5.0, 3.0, 1.0], start=1):
        tr.add(TraceRecord(1, k, d, 0.0, d, 0.1 * k))
    warm = LossTrace([TraceRecord(0, 1, 9.0, 0.0, 9.0, 0.1)])
    write_traces_csv(tmp_path / "t.csv", {"warm": warm, "frame_1": tr})
    back = read_traces_csv(tmp_path / "t.csv")
    assert set(back) == {0, 1} and [r.total for r in back[1].records] == [5.0, 3.0, 1.0]
    assert tr.iterations_to(1.0) == 3
    write_timing_csv(tmp_path / "s.csv", {"warm": 1.5, "frame_1": 0.5, "frame_2": 0.25})
    rows = read_timing_csv(tmp_path / "s.csv")
    assert [r[0] for r in rows] == ["warm", "frame_1", "frame_2"] and rows[-1][2] == pytest.approx(2.25)


def test_reference_network_engine_fields():
    """NetworkConfig maps onto the engine's FastResUNet3D program (ABI 3 desc fields)."""
    from paper_2507_14046_b200 import NetworkConfig
    from paper_2507_14046_b200 import _native as N
    from paper_2507_14046_b200.engine import net_fields
    f = net_fields(NetworkConfig(base_channels=8, use_depthwise=False, aspp_dilations=(1, 3)))
    assert f["arch"] == N.ARCH_FAST_RESUNET and f["channels"] == (8, 16, 32, 64)
    assert f["in_channels"] == 1 and f["depthwise"] == 0 and f["dilations"] == (1, 3)
    with pytest.raises(ValueError):
        net_fields(NetworkConfig(base_channels=6))  # channels must stay multiples of 4
    assert param_schema(NetworkConfig())[0].name == "stem.0.weight"
    names = [n for n, _ in N.NetDesc._fields_]
    assert names[-4:] == ["arch", "depthwise", "n_dil", "dil"]


# names the reference exports for the DIP path (pkg/src/d2ip/__init__.py:15-48) plus the
# priornet / pipeline functions SURVEY §8(b) lists (priornet.py:285-317, pipeline.py:341-391)
REFERENCE_DIP_NAMES = [
    "GridGeometry", "vectorize", "devectorize",
    "SensitivityMatrix", "VoltageFrame", "VoltageSequence", "assemble_sensitivity", "forward_project",
    "normalize_sensitivity",
    "FrameHistory", "TVWeights", "decay_weight", "spatial_tv", "temporal_tv", "tv4d",
    "NetworkConfig", "NoiseInput", "ParameterState", "init_parameters", "sample_noise_input",
    "build_model", "extract_parameters", "load_parameters", "forward_volume", "save_checkpoint", "load_checkpoint",
    "ReconstructionResult", "RunConfig", "ablation_mode", "reconstruct_frame", "reconstruct_sequence",
    "upws_pretrain", "loss", "predict_measurements",
]


def test_reference_dip_path_names_exported():
    import paper_2507_14046_b200 as D
    missing = [n for n in REFERENCE_DIP_NAMES if not callable(getattr(D, n, None))]
    assert not missing, missing
