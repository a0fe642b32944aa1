"""Pin the FastResUNet3D oracle (oracle/refnet.py) and the host-side parameter
schema / init / noise against the REAL reference backbone (tests/golden/
refnet.npz, written by tests/golden/make_golden_refnet.py from the unpatched
d2ip package, `priornet.py:96-293`)."""

import numpy as np
import pytest
import torch

from conftest import GOLDEN
from oracle import OracleFrameOptimizer, build_oracle_refnet
from paper_2507_14046_b200 import workloads as W
from paper_2507_14046_b200.priornet import (
    NetworkConfig,
    count_parameters,
    init_parameters,
    kaiming_flat,
    param_schema,
    sample_noise_input,
)

VARIANTS = {"dw4": dict(base_channels=4, use_depthwise=True, seed=1),
            "dense4": dict(base_channels=4, use_depthwise=False, seed=1),
            "dw8": dict(seed=1)}


def sha(a):
    import hashlib
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def relerr(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30))


@pytest.fixture(scope="module")
def gold():
    torch.set_num_threads(1)
    g = np.load(GOLDEN / "refnet.npz")
    wl = W.make_workload(W.small_spec(), seed=0)
    return g, wl


def test_harness_reproduces_refnet_inputs(gold):
    g, wl = gold
    assert sha(wl.matrix.values) == str(g["J_sha"])
    assert sha(wl.voltages.frames[0].values) == str(g["dv_sha"])
    assert sample_noise_input(wl.grid, 0).sha256() == str(g["z_sha"])


@pytest.mark.parametrize("tag", sorted(VARIANTS))
def test_schema_and_init_match_reference(gold, tag):
    g, _ = gold
    cfg = NetworkConfig(**VARIANTS[tag])
    assert init_parameters(cfg).checksum() == str(g[f"{tag}_theta0_sha"])
    assert count_parameters(cfg) == g[f"{tag}_l2sq_grads"].size
    if f"{tag}_theta0" in g:
        np.testing.assert_array_equal(kaiming_flat(cfg).numpy(), g[f"{tag}_theta0"])


def _runner(g, wl, tag, **kw):
    v = VARIANTS[tag]
    net = build_oracle_refnet(v.get("base_channels", 8), v.get("use_depthwise", True))
    J = wl.matrix.dense().values
    r = OracleFrameOptimizer(None, 1, g["z"], J, np.arange(J.shape[1]), tuple(g["output_map"]), 1e-3,
                             model=net, **kw)
    r.load(kaiming_flat(NetworkConfig(**v)))
    return r


@pytest.mark.parametrize("tag,mode", [("dw4", "l2sq"), ("dw4", "l2"), ("dense4", "l2sq"), ("dense4", "l2"),
                                      ("dw8", "l2sq")])
def test_oracle_refnet_grads_match_reference(gold, tag, mode):
    g, wl = gold
    r = _runner(g, wl, tag, data_norm=mode)
    total, data, reg, grads, _ = r.grads(g["dv"])
    assert data == pytest.approx(float(g[f"{tag}_{mode}_data"]), rel=1e-6)
    flat = torch.cat([v.reshape(-1) for v in grads.values()]).numpy()
    # the oracle's SE pool is x.mean (reference: AdaptiveAvgPool3d): fp32 ordering only
    assert relerr(flat, g[f"{tag}_{mode}_grads"]) < 1e-5


@pytest.mark.parametrize("tag", ["dw4", "dense4"])
def test_oracle_refnet_tv_grads_match_reference(gold, tag):
    g, wl = gold
    r = _runner(g, wl, tag, data_norm="l2", tv=(0.002, 1.0, 0.1, 1e-8))
    hist = [torch.as_tensor(h) for h in g["tv_history"]]
    total, data, reg, grads, _ = r.grads(g["dv"], hist)
    assert reg == pytest.approx(float(g[f"{tag}_tv_reg"]), rel=1e-5)
    assert total == pytest.approx(float(g[f"{tag}_tv_total"]), rel=1e-6)
    flat = torch.cat([v.reshape(-1) for v in grads.values()]).numpy()
    assert relerr(flat, g[f"{tag}_tv_grads"]) < 1e-5


@pytest.mark.parametrize("tag", ["dw4", "dense4"])
def test_oracle_refnet_ten_steps_match_reference(gold, tag):
    g, wl = gold
    r = _runner(g, wl, tag)
    vol, _, trace = r.optimize(g["dv"], [], 10, 0)
    got = np.array([[t[1], t[2], t[4]] for t in trace])
    np.testing.assert_allclose(got, g[f"{tag}_trace10"], rtol=1e-4)
    assert relerr(r.flat().numpy(), g[f"{tag}_theta10"]) < 1e-4
    np.testing.assert_allclose(vol, g[f"{tag}_volume10"], rtol=0, atol=1e-5)


def test_refnet_schema_names_follow_state_dict(gold):
    names = [e.name for e in param_schema(NetworkConfig())]
    assert names[:4] == ["stem.0.weight", "stem.0.bias", "stem.1.weight", "stem.1.bias"]
    assert "enc_block.0.conv1.0.weight" in names and "bottleneck.branches.2.weight" in names
    assert names[-2:] == ["tail.weight", "tail.bias"]
