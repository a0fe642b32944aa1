"""The drop-in names of the reference's DIP path (`pkg/src/d2ip/__init__.py:15-48`,
`priornet.py:285-317`, `forward.py:115-122`, `regularizers.py:86-140`) called
through the B200 package, each checked against the CPU oracle / numpy."""

import numpy as np
import pytest
import torch

import paper_2507_14046_b200 as D
from oracle import build_oracle_net
from oracle.frame import oracle_tv4d
from paper_2507_14046_b200 import workloads as W
from paper_2507_14046_b200.priornet import kaiming_flat, param_schema, sample_noise_input, state_from_flat

pytestmark = pytest.mark.gpu


def _vol(seed, shape=(12, 10, 8)):
    return np.random.default_rng(seed).normal(scale=0.1, size=shape).astype(np.float32)


@pytest.mark.parametrize("n_hist", [0, 1, 3])
def test_tv_functionals_vs_oracle(n_hist):
    cur = _vol(0)
    hist = [_vol(10 + k) for k in range(n_hist)]
    w = D.TVWeights()
    # numpy in -> float out (regularizers.py:94, 130, 139)
    ref_s = float(oracle_tv4d([], torch.as_tensor(cur), 1.0, 0.0, w.epsilon))
    assert isinstance(D.spatial_tv(cur), float)
    assert D.spatial_tv(cur) == pytest.approx(ref_s, rel=1e-5)
    ref = float(oracle_tv4d([torch.as_tensor(h) for h in hist], torch.as_tensor(cur), w.lambda_s, w.lambda_t,
                            w.epsilon))
    assert D.tv4d(hist, cur, w) == pytest.approx(ref, rel=1e-5)
    t = D.temporal_tv(hist, cur)
    if n_hist == 0:
        assert t == 0.0
    else:
        ref_t = float(oracle_tv4d([torch.as_tensor(h) for h in hist], torch.as_tensor(cur), 0.0, 1.0, w.epsilon))
        assert t == pytest.approx(ref_t, rel=1e-5)
    # tensor in -> tensor out with the gradient w.r.t. current (autograd)
    x = torch.tensor(cur, requires_grad=True)
    v = D.tv4d([torch.as_tensor(h) for h in hist], x, w)
    assert torch.is_tensor(v) and v.device == x.device
    (3.0 * v).backward()
    xr = torch.tensor(cur, requires_grad=True)
    vr = oracle_tv4d([torch.as_tensor(h) for h in hist], xr, w.lambda_s, w.lambda_t, w.epsilon)
    (3.0 * vr).backward()
    assert float(v) == pytest.approx(float(vr), rel=1e-5)
    assert float((x.grad - xr.grad).norm() / xr.grad.norm()) < 1e-5
    with pytest.raises(ValueError):
        D.spatial_tv(cur[0])


def test_forward_project_fp64():
    spec = W.CONFIGS["cfg0"]
    wl = W.make_workload(spec, seed=0, frames=1)
    q = np.random.default_rng(1).normal(size=wl.matrix.n_voxels)
    dense = wl.matrix.dense()
    ref = dense.values @ q
    y = D.forward_project(dense, q)
    assert y.dtype == np.float64 and y.shape == (dense.n_measurements,)
    assert np.max(np.abs(y - ref)) <= 1e-12 * np.max(np.abs(ref))
    ym = D.forward_project(wl.matrix, q)  # masked block: its masked columns of q
    assert np.max(np.abs(ym - ref)) <= 1e-6 * np.max(np.abs(ref))
    with pytest.raises(ValueError):
        D.forward_project(dense, q[:-1])


def test_build_model_extract_load_forward_volume():
    spec = W.small_spec()
    net = spec.network(seed=5)
    grid = spec.geometry()
    noise = sample_noise_input(grid, 3, spec.in_channels, 0.1)
    theta0 = D.init_parameters(net)
    model = D.build_model(net, grid.shape)
    assert list(model.state_dict()) == [e.name for e in param_schema(net)]
    D.load_parameters(model, theta0)
    st = D.extract_parameters(model, iteration_counter=7, provenance="upws")
    assert st.checksum() == theta0.checksum() and st.iteration_counter == 7 and st.provenance == "upws"
    out = model(noise.values)
    assert tuple(out.shape) == grid.shape and out.is_cuda
    oracle = build_oracle_net(spec.channels, spec.in_channels, seed=5)
    with torch.no_grad():
        ref = oracle(torch.tensor(noise.values, dtype=torch.float32)).numpy()
    assert np.max(np.abs(out.cpu().numpy() - ref)) < 1e-5
    vol = D.forward_volume(net, theta0, noise)
    assert vol.dtype == np.float64 and np.max(np.abs(vol - ref)) < 1e-5
    # the reference's own backbone through the same surface
    fnet = D.NetworkConfig(base_channels=4, seed=2)
    fn = sample_noise_input(grid, 0)
    fv = D.forward_volume(fnet, D.init_parameters(fnet), fn)
    assert fv.shape == grid.shape and np.isfinite(fv).all() and 0.0 < fv.min() <= fv.max() < 1.0


def test_device_J_cache_reused_across_standalone_calls():
    from paper_2507_14046_b200 import engine as E
    spec = W.small_spec(grid=(8, 8, 8), channels=(8, 16), in_channels=4, rings=(0.5,), frames=2)
    wl = W.make_workload(spec, seed=0)
    cfg = D.RunConfig(iters_warm=3, iters_first=2, iters_next=2, network=spec.network(), output_map=wl.output_map,
                      data_norm="l2sq", tv_weights=D.TVWeights(lambda_tv=0.0))
    noise = sample_noise_input(wl.grid, 0, 4, 0.1)
    E.clear_J_cache()
    th, _ = D.upws_pretrain(wl.matrix, wl.voltages.frames[0].values, noise, cfg)
    assert len(E._J_CACHE) == 1
    (J1,) = [e[1] for e in E._J_CACHE.values()]
    D.reconstruct_frame(th, wl.matrix, wl.voltages.frames[1].values, [], 2, cfg, noise)
    assert len(E._J_CACHE) == 1 and next(iter(E._J_CACHE.values()))[1] is J1


def test_reconstruct_sequences_batched_equals_single_runs():
    spec = W.small_spec(grid=(8, 8, 8), channels=(8, 16), in_channels=4, rings=(0.5,), frames=3)
    wls = [W.make_workload(spec, seed=s) for s in range(3)]
    cfg = D.RunConfig(iters_warm=6, iters_first=3, iters_next=2, learning_rate=1e-3, seed=10,
                      network=spec.network(), output_map=(-0.6, 0.3), data_norm="l2sq",
                      tv_weights=D.TVWeights(lambda_tv=0.0), precision="fp32")
    res = D.reconstruct_sequences_batched([w.matrix for w in wls], [w.voltages for w in wls], cfg, wls[0].grid)
    assert [r.index for r in res] == [0, 1, 2] and [r.seed for r in res] == [10, 11, 12]
    for r, w in zip(res, wls):
        one = D.reconstruct_sequence(w.matrix, w.voltages, D.RunConfig(**{**cfg.__dict__, "seed": r.seed}), w.grid)
        np.testing.assert_array_equal(r.sequence.values, one.sequence.values)
