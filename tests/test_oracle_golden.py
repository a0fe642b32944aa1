"""Pin the CPU oracle against the reference's own outputs (tests/golden/*.npz,
written by tests/golden/make_golden.py from the real d2ip package)."""

import numpy as np
import pytest
import torch

from conftest import GOLDEN
from oracle import OracleFrameOptimizer, build_oracle_net, oracle_reconstruct_sequence
from oracle.resunet import kaiming_reset
from paper_2507_14046_b200 import workloads as W
from paper_2507_14046_b200.priornet import sample_noise_input


def sha(a):
    import hashlib
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def relerr(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30))


@pytest.fixture(scope="module")
def cfg0():
    torch.set_num_threads(1)
    g = np.load(GOLDEN / "cfg0_step.npz")
    spec = W.CONFIGS["cfg0"]
    wl = W.make_workload(spec, seed=0)
    noise = sample_noise_input(wl.grid, 0, spec.in_channels, 0.1)
    return g, spec, wl, noise


def test_harness_reproduces_golden_inputs(cfg0):
    g, spec, wl, noise = cfg0
    assert sha(wl.matrix.values) == str(g["J_sha"])
    assert sha(wl.voltages.frames[0].values) == str(g["dv_sha"])
    assert noise.sha256() == str(g["z_sha"])


def test_oracle_kaiming_matches_reference_init(cfg0):
    g, spec, wl, noise = cfg0
    net = build_oracle_net(spec.channels, spec.in_channels, seed=1)
    flat = torch.cat([v.reshape(-1) for v in net.state_dict().values()]).numpy()
    np.testing.assert_array_equal(flat, g["theta0"])


def _runner(g, spec, wl, noise, dense=True, **kw):
    # dense=True feeds the reference's own operator form (zero columns outside the
    # mask): the oracle then reproduces the reference bit for bit.
    if dense:
        J = wl.matrix.dense().values
        cols = np.arange(J.shape[1])
    else:
        J, cols = wl.matrix.values, wl.matrix.columns_q()
    r = OracleFrameOptimizer(spec.channels, spec.in_channels, noise.values, J, cols,
                             tuple(g["output_map"]), 1e-3, **kw)
    r.load(g["theta0"])
    return r


@pytest.mark.parametrize("mode", ["l2sq", "l2"])
def test_oracle_step_grads_match_reference(cfg0, mode):
    g, spec, wl, noise = cfg0
    r = _runner(g, spec, wl, noise, data_norm=mode)
    total, data, reg, grads, _ = r.grads(g["dv"])
    assert data == float(g[f"{mode}_data"])
    flat = torch.cat([v.reshape(-1) for v in grads.values()]).numpy()
    np.testing.assert_array_equal(flat, g[f"{mode}_grads"])
    # compact masked J: same operator, different fp32 summation order
    rc = _runner(g, spec, wl, noise, dense=False, data_norm=mode)
    _, data_c, _, grads_c, _ = rc.grads(g["dv"])
    assert data_c == pytest.approx(float(g[f"{mode}_data"]), rel=1e-5)
    assert relerr(torch.cat([v.reshape(-1) for v in grads_c.values()]).numpy(), g[f"{mode}_grads"]) < 1e-5


def test_oracle_tv_grads_match_reference(cfg0):
    g, spec, wl, noise = cfg0
    r = _runner(g, spec, wl, noise, data_norm="l2", tv=(0.002, 1.0, 0.1, 1e-8))
    hist = [torch.as_tensor(h, dtype=torch.float32) for h in g["tv_history"]]
    total, data, reg, grads, _ = r.grads(g["dv"], hist)
    assert reg == float(g["tv_reg"])
    assert total == float(g["tv_total"])
    flat = torch.cat([v.reshape(-1) for v in grads.values()]).numpy()
    np.testing.assert_array_equal(flat, g["tv_grads"])


@pytest.mark.parametrize("k", [1, 10])
def test_oracle_adam_trajectory_matches_reference(cfg0, k):
    g, spec, wl, noise = cfg0
    r = _runner(g, spec, wl, noise)
    vol, mapped, trace = r.optimize(g["dv"], [], k, 0)
    np.testing.assert_array_equal(r.flat().numpy(), g[f"theta{k}"])
    np.testing.assert_array_equal([t[2] for t in trace], g[f"trace{k}"][:, 1])
    np.testing.assert_array_equal(vol, g[f"volume{k}"])


@pytest.mark.slow
def test_oracle_cfg0_full_run_matches_reference(cfg0):
    g, spec, wl, noise = cfg0
    torch.set_num_threads(1)
    r = _runner(g, spec, wl, noise)
    vol, mapped, trace = r.optimize(g["dv"], [], 300, 0)
    np.testing.assert_array_equal([t[2] for t in trace], g["trace300"][:, 1])
    np.testing.assert_array_equal(vol, g["volume300"])


def test_oracle_sequence_matches_reference():
    g = np.load(GOLDEN / "seq_mini.npz")
    spec = W.small_spec()
    wl = W.make_workload(spec, seed=0)
    noise = sample_noise_input(wl.grid, 1, spec.in_channels, 0.1)
    assert noise.sha256() == str(g["z_sha"])
    np.testing.assert_array_equal(
        torch.cat([v.reshape(-1) for v in build_oracle_net(spec.channels, 8, seed=2).state_dict().values()]).numpy(),
        g["theta0"])
    torch.set_num_threads(1)
    d = wl.matrix.dense().values
    res = oracle_reconstruct_sequence(spec.channels, spec.in_channels, noise.values, d,
                                      np.arange(d.shape[1]), [f.values for f in wl.voltages.frames],
                                      g["theta0"], tuple(g["output_map"]), 12, 6, 4, 1e-3)
    assert [c[0] for c in res["chain"]] == list(g["provenance"])
    assert [r[2] for r in res["records"]] == list(g["iterations"])
    np.testing.assert_array_equal(res["columns"], g["values"])
    np.testing.assert_array_equal(res["final"].numpy(), g["theta_final"])
    for key in ("warm", "frame_1", "frame_4"):
        np.testing.assert_array_equal([t[2] for t in res["traces"][key]], g[f"trace_{key}"][:, 1])


def test_oracle_tv_sequence_matches_reference():
    g = np.load(GOLDEN / "seq_mini.npz")
    spec = W.small_spec()
    wl = W.make_workload(spec, seed=0)
    noise = sample_noise_input(wl.grid, 1, spec.in_channels, 0.1)
    torch.set_num_threads(1)
    d = wl.matrix.dense().values
    res = oracle_reconstruct_sequence(spec.channels, spec.in_channels, noise.values, d,
                                      np.arange(d.shape[1]), [f.values for f in wl.voltages.frames[:3]],
                                      g["theta0"], tuple(g["output_map"]), 12, 6, 4, 1e-3,
                                      data_norm="l2", tv=(0.002, 1.0, 0.1, 1e-8))
    np.testing.assert_array_equal(res["columns"], g["tv_values"])
    for key in ("warm", "frame_2", "frame_3"):
        np.testing.assert_array_equal([t[4] for t in res["traces"][key]], g[f"tvtrace_{key}"][:, 2])


# ---------------------------------------------------------------------------
# 4-level net (cfg2 / cfg4 topology) and the joint warm-start, pinned bit for bit


def _l4():
    g = np.load(GOLDEN / "level4.npz")
    spec = W.small_spec(name="l4", grid=(16, 16, 16), channels=tuple(int(c) for c in g["channels"]),
                        in_channels=4, rings=(0.3, 0.7), frames=1)
    wl = W.make_workload(spec, seed=2)
    noise = sample_noise_input(wl.grid, 2, spec.in_channels, 0.1)
    return g, spec, wl, noise


def test_oracle_level4_matches_reference():
    torch.set_num_threads(1)
    g, spec, wl, noise = _l4()
    assert sha(wl.matrix.values) == str(g["J_sha"]) and noise.sha256() == str(g["z_sha"])
    net = build_oracle_net(spec.channels, spec.in_channels, seed=int(g["net_seed"]))
    theta0 = torch.cat([v.reshape(-1) for v in net.state_dict().values()]).numpy()
    from paper_2507_14046_b200.priornet import kaiming_flat, param_schema, state_from_flat
    cfgn = spec.network(seed=int(g["net_seed"]))
    np.testing.assert_array_equal(kaiming_flat(cfgn).numpy(), theta0)
    assert state_from_flat(torch.from_numpy(theta0), param_schema(cfgn)).checksum() == str(g["theta0_sha"])
    J = wl.matrix.dense().values
    r = OracleFrameOptimizer(spec.channels, spec.in_channels, noise.values, J, np.arange(J.shape[1]),
                             tuple(g["output_map"]), 1e-3)
    r.load(theta0)
    _, data, _, grads, _ = r.grads(g["dv"])
    assert data == float(g["l2sq_data"])
    np.testing.assert_array_equal(torch.cat([v.reshape(-1) for v in grads.values()]).numpy(), g["l2sq_grads"])
    r.load(theta0)
    r.optimize(g["dv"], [], 5, 0)
    np.testing.assert_array_equal(r.flat().numpy(), g["theta5"])


def test_oracle_joint_mean_frame_upws_matches_reference():
    """The reference's upws_pretrain(dv0 = mean of the frames) is reproduced bit for bit."""
    torch.set_num_threads(1)
    g = np.load(GOLDEN / "joint_upws.npz")
    spec = W.small_spec(grid=(8, 8, 8), channels=(8, 16), in_channels=4, rings=(0.5,), frames=4)
    wl = W.make_workload(spec, seed=0)
    np.testing.assert_array_equal(np.stack([f.values for f in wl.voltages.frames]), g["dvs"])
    noise = sample_noise_input(wl.grid, 0, 4, 0.1)
    J = wl.matrix.dense().values
    r = OracleFrameOptimizer(spec.channels, spec.in_channels, noise.values, J, np.arange(J.shape[1]),
                             tuple(g["output_map"]), 1e-3)
    r.load(g["theta0"])
    r.optimize(g["dvs"].mean(0), [], 10, 0)
    np.testing.assert_array_equal(r.flat().numpy(), g["theta10"])


def test_cfg1_band_fixture_is_consistent():
    """tests/golden/seq_cfg1_band.npz (make_band_cfg1.py: the oracle at other host thread counts)
    holds distinct reorderings of the cfg1-budget run, and its 8-thread member reproduces the band
    of seq_cfg1.npz (written beside the real reference's run) bit for bit."""
    gq = np.load(GOLDEN / "seq_cfg1.npz")
    gb = np.load(GOLDEN / "seq_cfg1_band.npz")
    members = {k: gb[k] for k in gb.files if k.startswith("values_t")}
    assert set(members) == {"values_t2", "values_t4", "values_t8"}
    for v in members.values():
        assert v.shape == gq["values"].shape and np.isfinite(v).all()
    np.testing.assert_array_equal(members["values_t8"], gq["band_values"])
    assert not np.array_equal(members["values_t2"], members["values_t4"])
    assert not np.array_equal(members["values_t4"], members["values_t8"])
