"""Benchmark of the DIP step (BASELINE.json metric "DIP iters/sec & tsEIT frames/sec").

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload cfg1] [--impl reference]

A step is one DIP iteration (ResUNet forward + masked J.sigma data term +
adjoint + backward + Adam) of the workload, replayed from a CUDA graph with
every input resident in HBM. N=1 runs BASELINE configs[1] (cfg1: 32^3 grid,
16/32/64 ResUNet, M=928, V=25,984, TF32 convolutions). The single-sequence
workloads do not shard (the TPP chain is sequential), so N>1
runs N independent replicas (one sequence per rank, weak scaling) and `value`
is the total iterations of all ranks / the max over ranks of the device time.

`e2e` is the same metric through the public API: one `reconstruct_sequence`
call on host (numpy) inputs at the workload's budgets, host->device uploads of
J / Z / dv and device->host reads of traces, checksums and volumes inside the
timed region.

`--impl reference` times the reference algorithm's CPU implementation (the
oracle port, `oracle/`, bit-exact to the reference package on the golden
cases) on the box's host cores, same metric and config.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

PEAKS_PATH = ROOT / "MEASURED_PEAKS.json"
FALLBACK = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}


def peaks():
    try:
        d = json.loads(PEAKS_PATH.read_text())
        return d, "measured"
    except Exception:
        return FALLBACK, "fallback"


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


class Clocks:
    """nvidia-smi sampling during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.path = Path(f"/tmp/d2ip_clocks_{os.getpid()}.csv")

    def __enter__(self):
        try:
            self.fh = open(self.path, "w")
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "50"],
                                         stdout=self.fh, stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *a):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
            self.fh.close()

    def summary(self):
        if self.proc is None or not self.path.exists():
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        rows = [r.split(", ") for r in self.path.read_text().strip().splitlines() if r.strip()]
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in rows:
            try:
                sm.append(float(r[1]))
                mx = float(r[2])
                for n, v in zip(names, r[5:9]):
                    if v.strip().lower() == "active":
                        reasons.add(n)
            except (ValueError, IndexError):
                continue
        loaded = [s for s in sm if mx and s > 0.5 * mx] or sm
        return {"sm_mhz": statistics.median(loaded) if loaded else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


# ---------------------------------------------------------------------------


def algorithmic_units(spec, net, M, Vp):
    """Per-iteration algorithmic bytes / FLOPs."""
    from paper_2507_14046_b200.priornet import param_schema

    R, C, P = spec.grid
    ch, cz = spec.channels, spec.in_channels
    L = len(ch)
    V = [R * C * P >> (3 * l) for l in range(L)]
    flops = 0.0

    def conv(cin, cout, k, vout, dgrad=True):
        f = 2.0 * k ** 3 * cin * cout * vout
        return f * (3 if dgrad else 2)

    flops += conv(cz, ch[0], 3, V[0], dgrad=False)
    for i in range(1, L):
        flops += conv(ch[i - 1], ch[i], 3, V[i]) + conv(ch[i], ch[i], 3, V[i]) + conv(ch[i - 1], ch[i], 1, V[i])
    flops += conv(ch[L - 1], ch[L - 1], 3, V[L - 1]) * 2 + conv(ch[L - 1], ch[L - 1], 1, V[L - 1])
    for l in range(L - 2, -1, -1):
        cin = ch[l + 1] + ch[l]
        flops += conv(cin, ch[l], 3, V[l]) + conv(ch[l], ch[l], 3, V[l]) + conv(cin, ch[l], 1, V[l])
    flops += conv(ch[0], 1, 3, V[0])
    nparams = sum(e.numel for e in param_schema(net))
    return {"conv_flops": flops, "jac_bytes_per_pass": 4.0 * M * Vp + 4.0 * Vp, "adam_bytes": 28.0 * nparams,
            "n_params": nparams}


def time_kernel(fn, reps=20, warm=3):
    import torch

    for _ in range(warm):
        fn()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    s.record()
    for _ in range(reps):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / reps / 1e3


def run_gpu(args):
    import torch
    import torch.distributed as dist
    import ctypes as C

    from paper_2507_14046_b200 import _native as N
    from paper_2507_14046_b200 import workloads as W
    from paper_2507_14046_b200.engine import DeviceNet
    from paper_2507_14046_b200.priornet import kaiming_flat, sample_noise_input

    ws, rank, local = dist_env()
    torch.cuda.set_device(local)
    if ws > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    spec = W.CONFIGS[args.workload]
    seed = rank
    if spec.sequences > 1:
        # cfg3: this rank's share of the independent sequences, batched in lockstep
        from paper_2507_14046_b200.distributed import shard
        mine = list(shard(spec.sequences, ws, rank))
        wl = W.make_workload(spec, seed=mine[0], frames=1)
        net = spec.network()
        dn = DeviceNet(net, wl.grid.shape, wl.matrix.n_measurements, wl.matrix.mask, batch=len(mine),
                       j_shared=False, data_norm="l2sq", output_map=wl.output_map, lr=spec.learning_rate,
                       precision=args.precision or spec.precision, max_iters=args.warmup + args.steps + 8)
        for b, s in enumerate(mine):
            Jd, _ = W.jacobian_device(spec, s)
            dn.set_J_device(Jd, b=b)
            del Jd
            dn.set_noise(sample_noise_input(wl.grid, s, spec.in_channels, 0.1).values, b=b)
            dn.set_theta(kaiming_flat(net, seed=s + 1), b=b)
            dn.set_dv(wl.voltages.frames[0].values, b=b)
        units_per_step = len(mine)
    elif spec.n_measurements * int(np.prod(spec.grid)) > 64 * 1024 * 1024:
        # cfg2 / cfg4: J (GB-sized) synthesised on the GPU, never on the host
        J_dev, mask, dv_dev, omap = W.device_frame(spec, seed)
        wl = None
        net = spec.network(seed=seed + 1)
        grid = spec.geometry()
        noise = sample_noise_input(grid, seed, spec.in_channels, 0.1)
        dn = DeviceNet(net, grid.shape, J_dev.shape[0], mask, data_norm="l2sq", output_map=omap,
                       lr=spec.learning_rate, precision=args.precision or spec.precision,
                       max_iters=args.warmup + args.steps + 8)
        dn.set_noise(noise.values)
        dn.set_J_device(J_dev)
        del J_dev
        dn.set_theta(kaiming_flat(net))
        dn.dv[0, 0].copy_(dv_dev)
        units_per_step = 1
    else:
        wl = W.make_workload(spec, seed=seed, frames=min(spec.frames, 20))
        net = spec.network(seed=seed + 1)
        noise = sample_noise_input(wl.grid, seed, spec.in_channels, 0.1)
        if args.net == "fast":  # the reference's own backbone on this workload (1-channel U[0,1) noise)
            from paper_2507_14046_b200.priornet import NetworkConfig
            net = NetworkConfig(base_channels=args.base_channels, use_depthwise=not args.dense, seed=seed + 1)
            noise = sample_noise_input(wl.grid, seed)
        dn = DeviceNet(net, wl.grid.shape, wl.matrix.n_measurements, wl.matrix.mask, data_norm="l2sq",
                       output_map=wl.output_map, lr=spec.learning_rate,
                       precision=args.precision or spec.precision, max_iters=args.warmup + args.steps + 8)
        dn.set_noise(noise.values)
        dn.set_J_host(wl.matrix.values)
        dn.set_theta(kaiming_flat(net))
        dn.set_dv(wl.voltages.frames[0].values)
        units_per_step = 1
    dn.reset_frame()
    torch.cuda.synchronize()
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    for _ in range(args.warmup):
        dn.run(1)
    torch.cuda.synchronize()
    if ws > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with Clocks(local) as clk:
        for i in range(args.steps):
            flush.zero_()  # L2 flush between timed iterations (outside the events)
            ev[i][0].record()
            dn.run(1)
            ev[i][1].record()
        torch.cuda.synchronize()
    t_dev = sum(a.elapsed_time(b) for a, b in ev) / 1e3
    if ws > 1:
        t = torch.tensor([t_dev], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        t_dev = float(t.item())
        dist.barrier()
    status = dn.status_host()
    assert status[0, 1] == 0, "non-finite loss during the benchmark"
    launches = dn.launches_per_iter()
    its = ws * units_per_step * args.steps / t_dev

    # --- no-flush steady state (informational): J may stay L2-resident
    torch.cuda.synchronize()
    s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s0.record()
    dn.run(args.steps)
    s1.record()
    torch.cuda.synchronize()
    its_hot = units_per_step * args.steps / (s0.elapsed_time(s1) / 1e3)

    # --- roofline of the dominant kernels, timed live on this stream
    pk, pk_kind = peaks()
    units = algorithmic_units(spec, net, dn.M, dn.Vp) if args.net == "config" else {
        "conv_flops": float("nan"), "n_params": dn.n_params}
    L = N.lib()
    st = C.c_void_p(torch.cuda.current_stream().cuda_stream)
    t_flush = time_kernel(lambda: flush.zero_())

    def jac_probe(M, Vp, J):
        nseg = L.d2ip_jac_nseg(Vp)
        part = torch.empty(M * nseg, device="cuda")
        sig = torch.randn(Vp, device="cuda")

        def run():
            flush.zero_()
            N.check(L.d2ip_jac_fwd(C.c_void_p(J.data_ptr()), 0, C.c_void_p(sig.data_ptr()), 0, M, Vp,
                                   C.c_void_p(part.data_ptr()), nseg, 1, st), "jac_fwd")
        t = max(time_kernel(run) - t_flush, 1e-9)
        byt = 4.0 * M * Vp + 4.0 * Vp
        return {"bound": "hbm", "kernel": "jac_fwd (K5, J.sigma GEMV)", "M": M, "Vp": Vp,
                "achieved": round(byt / t / 1e9, 1), "peak": pk["hbm_gbs"], "unit": "GB/s",
                "frac": round(byt / t / 1e9 / pk["hbm_gbs"], 4), "algorithmic_bytes_per_launch": byt,
                "avg_launch_s": t, "peak_source": pk_kind,
                "note": "read-only stream vs the copy (read+write) peak, so frac can exceed 1; "
                        f"vs the 8,000 GB/s nominal: {byt / t / 8e12:.3f}"}

    jac_cfg = jac_probe(dn.M, dn.Vp, dn.J)
    # the same kernel on cfg2's 3,904 x 103,296 operator (1.6 GB, far beyond L2)
    hbm_probe = None
    if not args.skip_probe:
        Vp2 = (103296 + 3) // 4 * 4
        J2 = torch.randn(3904, Vp2, device="cuda")
        hbm_probe = jac_probe(3904, Vp2, J2)
        del J2
    # dominant kernel: the tcgen05 conv on cfg1's largest layer (dec0.conv1,
    # 48 -> 16 channels at 32^3), one launch timed live through the C ABI
    conv_roof = conv_probe(L, N, C, st, pk, pk_kind, flush, t_flush) if spec.channels[0] == 16 and args.net == "config" else None
    # the bf16 tensor-core kernels on cfg4's largest layer (dec0.conv1, 96 -> 32 at 96x96x48)
    conv_bf16 = None if args.skip_probe else conv_bf16_probe(L, N, C, st, flush, t_flush)
    # K7 Adam on cfg4's flat parameter buffer (9.53 M parameters, 28 B each per step)
    adam_roof = None
    if not args.skip_probe:
        n_ad = 9_529_233
        bufs = [torch.randn(n_ad, device="cuda") for _ in range(4)]
        bufs[3].abs_()
        stepv = torch.ones(1, dtype=torch.int32, device="cuda")

        def adam_run():
            flush.zero_()
            N.check(L.d2ip_adam(*[C.c_void_p(b.data_ptr()) for b in bufs], n_ad, 1e-3, 0.9, 0.999, 1e-8,
                                C.c_void_p(stepv.data_ptr()), st), "adam")
        t_ad = max(time_kernel(adam_run) - t_flush, 1e-9)
        byt = 28.0 * n_ad
        adam_roof = {"bound": "hbm", "kernel": "adam_k (K7, flat float4 Adam)", "n_params": n_ad,
                     "algorithmic_bytes_per_launch": byt, "avg_launch_s": t_ad,
                     "achieved": round(byt / t_ad / 1e9, 1), "peak": pk["hbm_gbs"], "unit": "GB/s",
                     "frac": round(byt / t_ad / 1e9 / pk["hbm_gbs"], 4), "peak_source": pk_kind,
                     "note": f"p, g, m, v read + p, m, v written; vs the 8,000 GB/s nominal: {byt / t_ad / 8e12:.3f}"}
        del bufs
    # whole-iteration tensor-throughput view of the convolutions
    conv_tflops = units["conv_flops"] * units_per_step / (t_dev / args.steps) / 1e12
    roofline = conv_roof or jac_cfg

    # --- e2e through the public API (rank-local, one full sequence)
    e2e = None
    if not args.skip_e2e and units_per_step == 1 and wl is not None and args.net == "config":
        e2e = run_e2e(spec, wl, args, ws)

    out = {
        "metric": "DIP iters/sec", "value": round(its, 2), "unit": "it/s", "n_gpus": ws, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(1e3 * t_dev / args.steps, 4), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": ("f32 (TF32-class convs: 3xbf16 hi/lo operand splits on kind::f16, fp32 accumulate)"
                  if os.environ.get("D2IP_TF32_BF3", "1") != "0" else "f32 (3xTF32 conv operands)")
                 if (args.precision or spec.precision) == "tf32" else
                 ("f32 (bf16 conv operands, fp32 accumulate)" if (args.precision or spec.precision) == "bf16" else "f32"),
        "data": "synthetic (seeded BASELINE cfg generator; random-init weights)",
        "config": {"workload": args.workload + ("" if args.net == "config" else
                                                f"+FastResUNet3D(b={args.base_channels},{'dense' if args.dense else 'depthwise'})"),
                   "grid": list(spec.grid), "channels": list(spec.channels),
                   "C_z": spec.in_channels, "M": dn.M, "V": dn.V, "n_params": units["n_params"],
                   "precision": args.precision or spec.precision,
                   "parallelism": f"replicas x{ws}" if ws > 1 else "single GPU",
                   "l2": "flushed between timed iterations (256 MB write)"},
        "frames_per_sec": round(its * spec.frames / (spec.iters_warm + spec.frames * spec.iters_next), 4),
        "its_no_flush": round(its_hot * ws, 2),
        "conv_tflops_effective": round(conv_tflops, 3),
        "gpu_launches": launches * args.steps,
        "launches_per_step": launches,
        "roofline": roofline,
        "roofline_jac_cfg": jac_cfg,
        "roofline_jac_hbm": hbm_probe,
        "roofline_conv_bf16_cfg4": conv_bf16,
        "roofline_adam_cfg4": adam_roof,
        "clocks": clk.summary(),
    }
    if units_per_step > 1:
        out["config"]["sequences_per_gpu"] = units_per_step
        out["config"]["parallelism"] = f"{spec.sequences} sequences sharded over {ws} GPU(s), batched in lockstep"
    if e2e is not None:
        out["e2e"] = e2e
    if rank == 0 and ws == 1 and not args.skip_cpu:
        out["cpu_baseline"] = cpu_baseline(args.workload, seconds=args.cpu_seconds)
    if rank == 0:
        print(json.dumps(out))
    if ws > 1:
        dist.destroy_process_group()


# dense TF32 tensor peak measured with tools/umma_rate.cu (148 SMs x 2 CTAs,
# M=128 N=256 kind::tf32 MMAs): 1104.5 TFLOP/s (profiles/r1_umma_rate.txt)
TF32_PEAK_TFLOPS = 1104.5


def conv_probe(L, N, C, st, pk, pk_kind, flush, t_flush):
    """One launch of the tcgen05 conv on cfg1's dec0.conv1 shape (48 -> 16 @ 32^3),
    timed with CUDA events; algorithmic FLOPs = 2*27*Cin*Cout*V."""
    import torch

    cin, cout, D = 48, 16, 32
    x = torch.randn(1, D, D, D, cin, device="cuda")
    y = torch.empty(1, D, D, D, cout, device="cuda")
    w = torch.randn(cout * cin * 27 + cout, device="cuda") * 0.05

    def act(t, c):
        a = N.Act()
        a.ptr, a.d, a.h, a.w, a.c, a.cstride = t.data_ptr(), D, D, D, c, c
        a.bstride = D * D * D * c
        return a

    wsn = L.d2ip_conv3d_ws_bytes(cin, cout, 3, 1, N.PREC["tf32"], 1)
    ws = torch.empty(wsn, dtype=torch.uint8, device="cuda")
    xa, ya = act(x, cin), act(y, cout)

    def run():
        flush.zero_()
        N.check(L.d2ip_conv3d_fwd(xa, C.c_void_p(w.data_ptr()), C.c_void_p(w.data_ptr() + 4 * cout * cin * 27), 0,
                                  3, 1, ya, 0, N.PREC["tf32"], C.c_void_p(ws.data_ptr()), wsn, 1, st), "conv")
    t = max(time_kernel(run) - t_flush, 1e-9)
    flops = 2.0 * 27 * cin * cout * D ** 3
    peak = pk.get("bf16_tflops", 1665.3)  # MEASURED_PEAKS.json: dense bf16 (the operand type the kernel runs)
    traffic = None  # DRAM bytes of this launch from the committed `ncu --set full` capture
    try:
        prof = json.loads((Path(__file__).resolve().parent / "profiles" / "r1_ncu_cfg1dec0c1.json").read_text())
        scale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
        traffic = sum(float(prof[k]["value"]) * scale[prof[k]["unit"]]
                      for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"))
    except Exception:
        traffic = None
    b3 = os.environ.get("D2IP_TF32_BF3", "1") != "0"
    # shape bound: an M=128 x N=16 MMA reads 4 KB (A) + 0.5 KB (B) of shared memory in ~39 cycles
    # (tools/umma_chains.cu): kind::f16 does 2*128*16*16 flop in it (of 8,192 flop/cycle/SM at
    # the 2,209 TFLOP/s probe peak), kind::tf32 half that; 3x MMAs per fp32-accurate product
    f16_probe = F16_PEAK_TFLOPS
    n16 = f16_probe * (2 * 128 * 16 * 16 / 39) / 8192 / 3 if b3 else TF32_PEAK_TFLOPS * (2 * 128 * 16 * 8 / 39) / 4096 / 3
    return {"bound": "tensor",
            "kernel": "conv_tc_k (K1, tcgen05 %s implicit GEMM) incl. weight pack" % ("3xbf16 kind::f16" if b3 else "3xTF32"),
            "layer": "dec0.conv1 48->16 @ 32^3", "achieved": round(flops / t / 1e12, 2), "peak": peak,
            "unit": "TFLOP/s", "frac": round(flops / t / 1e12 / peak, 4), "traffic": traffic,
            "traffic_source": "profiles/r1_ncu_cfg1dec0c1.json (ncu --set full, dram read+write bytes)",
            "algorithmic_flops_per_launch": flops, "avg_launch_s": t,
            "peak_source": "MEASURED_PEAKS.json bf16_tflops (cuBLAS 8192^3 burst); the kernel's pipe peak from "
                           "tools/umma_rate.cu is %.1f (kind::f16) / %.1f (kind::tf32) TFLOP/s" % (f16_probe, TF32_PEAK_TFLOPS),
            "n16_shape_bound": round(n16, 1),
            "n16_shape_bound_source": "16 output channels: M=128 x N=16 MMAs bound by shared-memory operand reads "
                                      "(39 cycles each, tools/umma_chains.cu), 3 MMAs per fp32-accurate product",
            "frac_of_n16_shape_bound": round(flops / t / 1e12 / n16, 4)}


# dense kind::f16 peak measured the same way (profiles/r1_umma_rate.txt): 2,209 TFLOP/s.
# At N = 32 output channels an M = 128 MMA reads 4 KB (A) + 1 KB (B) of shared
# memory in ~40 cycles (tools/umma_chains.cu), which caps it at 40 % of that peak.
F16_PEAK_TFLOPS = 2209.1
F16_N32_BOUND_TFLOPS = F16_PEAK_TFLOPS * (2 * 128 * 32 * 16 / 40) / 8192  # 3,277 of 8,192 flop/cycle/SM


def conv_bf16_probe(L, N, C, st, flush, t_flush):
    """bf16 (kind::f16) forward conv and weight gradient of cfg4's dec0.conv1 (96 -> 32
    channels at 96x96x48), inputs with their bf16 twins as in the engine; one launch
    each timed with CUDA events (weight pack included in the forward)."""
    import torch

    cin, cout, dims = 96, 32, (96, 96, 48)
    V = dims[0] * dims[1] * dims[2]
    x = torch.randn(1, *dims, cin, device="cuda")
    y = torch.randn(1, *dims, cout, device="cuda")
    xt, yt = x.to(torch.bfloat16), y.to(torch.bfloat16)
    w = torch.randn(cout * cin * 27 + cout, device="cuda") * 0.05
    gw = torch.zeros_like(w)

    def act(t, tw, c):
        a = N.Act()
        a.ptr, a.c, a.cstride = t.data_ptr(), c, c
        a.d, a.h, a.w = dims
        a.bstride = V * c
        a.bf16 = tw.data_ptr()
        return a

    xa, ya = act(x, xt, cin), act(y, yt, cout)
    wsn = L.d2ip_conv3d_ws_bytes(cin, cout, 3, 1, N.PREC["bf16"], 1)
    ws = torch.empty(wsn, dtype=torch.uint8, device="cuda")
    wgn = L.d2ip_conv3d_wgrad_ws_bytes(xa, ya, 3, 1)
    wgs = torch.empty(wgn, dtype=torch.uint8, device="cuda")

    def fwd():
        flush.zero_()
        N.check(L.d2ip_conv3d_fwd(xa, C.c_void_p(w.data_ptr()), C.c_void_p(w.data_ptr() + 4 * cout * cin * 27), 0,
                                  3, 1, act(y, yt, cout), 0, N.PREC["bf16"], C.c_void_p(ws.data_ptr()), wsn, 1, st),
                "conv bf16")

    def wgrad():
        flush.zero_()
        N.check(L.d2ip_conv3d_wgrad(xa, ya, 3, 1, C.c_void_p(gw.data_ptr()), 0, C.c_void_p(wgs.data_ptr()), wgn,
                                    N.PREC["bf16"], 1, st), "wgrad bf16")
    flops = 2.0 * 27 * cin * cout * V
    pk, _ = peaks()
    peak = pk.get("bf16_tflops", 1665.3)
    out = {"bound": "tensor", "layer": "cfg4 dec0.conv1 96->32 @ 96x96x48, bf16 operands (twins), fp32 accumulate",
           "algorithmic_flops_per_launch": flops, "unit": "TFLOP/s", "peak": peak,
           "peak_source": "MEASURED_PEAKS.json bf16_tflops (cuBLAS burst); tcgen05 kind::f16 probe peak %.1f" % F16_PEAK_TFLOPS,
           "n32_operand_bound": round(F16_N32_BOUND_TFLOPS, 1),
           "n32_operand_bound_source": "M=128 x N=32 MMA = 40 cycles of shared-memory operand reads "
                                       "(tools/umma_chains.cu); the layer's 32 output channels cap kind::f16 there"}
    for name, fn, kern in (("fwd", fwd, "conv_tc_k<bf16> (K1) incl. weight pack"),
                           ("wgrad", wgrad, "wgrad_bf_k (K3, kind::f16) incl. partial reduction")):
        t = max(time_kernel(fn) - t_flush, 1e-9)
        tf = flops / t / 1e12
        out[name] = {"kernel": kern, "avg_launch_s": t, "achieved": round(tf, 1),
                     "frac": round(tf / peak, 4), "frac_of_n32_bound": round(tf / F16_N32_BOUND_TFLOPS, 4)}
    del x, y, xt, yt, ws, wgs
    return out


def run_e2e(spec, wl, args, ws):
    import torch

    from paper_2507_14046_b200 import reconstruct_sequence
    from paper_2507_14046_b200 import workloads as W
    from paper_2507_14046_b200.forward import MaskedSensitivity, VoltageSequence

    frames = min(spec.frames, args.e2e_frames)
    volts = VoltageSequence(wl.voltages.frames[:frames])
    cfg = W.run_config_for(spec, wl.output_map, seed=wl.seed, precision=args.precision or spec.precision,
                           iters_warm=min(spec.iters_warm, args.e2e_warm))
    matrix = MaskedSensitivity(np.array(wl.matrix.values), wl.matrix.mask)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    res = reconstruct_sequence(matrix, volts, cfg, wl.grid)
    torch.cuda.synchronize()
    secs = time.perf_counter() - t0
    iters = cfg.iters_warm + sum(f.iterations for f in res.frame_records)
    h2d = matrix.values.nbytes + 4 * np.prod(wl.grid.shape) * spec.in_channels + frames * 4 * wl.matrix.n_measurements
    nparam = res.states["init"].flat().numel()
    # theta0 is uploaded once: every later stage starts from the theta the device already
    # holds (UPWS -> frame 1 -> TPP hand-off, pipeline.py:529)
    h2d += 4 * nparam
    # per stage: sigmoid volume (fp32) + exported theta + status; per iteration: trace row (4 fp32)
    d2h = (frames + 1) * (4 * np.prod(wl.grid.shape) + 4 * nparam + 16) + 4 * iters * 4
    return {"value": round(iters / secs, 2), "unit": "it/s", "h2d_bytes_per_step": int(h2d / iters),
            "d2h_bytes_per_step": int(d2h / iters), "call": "reconstruct_sequence",
            "iterations": int(iters), "frames": frames, "seconds": round(secs, 3),
            "frames_per_sec": round(frames / secs, 4)}


def cpu_baseline(workload: str, seconds: float = 15.0, threads: int | None = None):
    """The oracle port (bit-exact to the reference on the golden cases) timed on
    the host cores on a bounded sample of the same workload."""
    import torch

    from oracle import OracleFrameOptimizer
    from oracle.resunet import kaiming_reset
    from paper_2507_14046_b200 import workloads as W
    from paper_2507_14046_b200.priornet import sample_noise_input

    spec = W.CONFIGS[workload]
    wl = W.make_workload(spec, seed=0, frames=1)
    noise = sample_noise_input(wl.grid, 0, spec.in_channels, 0.1)
    threads = threads or os.cpu_count()
    prev = torch.get_num_threads()
    torch.set_num_threads(threads)
    try:
        r = OracleFrameOptimizer(spec.channels, spec.in_channels, noise.values, wl.matrix.values,
                                 wl.matrix.columns_q(), wl.output_map, spec.learning_rate)
        kaiming_reset(r.model, 1)
        dv = wl.voltages.frames[0].values
        r.optimize(dv, [], 1, 1)  # warm-up
        n, t = 0, 0.0
        while t < seconds and n < 200:
            t0 = time.perf_counter()
            r.optimize(dv, [], 1, 1)
            t += time.perf_counter() - t0
            n += 1
    finally:
        torch.set_num_threads(prev)
    return {"value": round(n / t, 4), "unit": "it/s", "cores": threads, "kind": "port",
            "sample": f"{n} DIP iterations of {workload} (oracle port of pipeline.py:310-331, torch CPU fp32)"}


def run_reference(args):
    ws, rank, local = dist_env()
    if rank != 0:
        return
    per = []
    import torch

    from oracle import OracleFrameOptimizer
    from oracle.resunet import kaiming_reset
    from paper_2507_14046_b200 import workloads as W
    from paper_2507_14046_b200.priornet import sample_noise_input

    spec = W.CONFIGS[args.workload]
    wl = W.make_workload(spec, seed=0, frames=1)
    noise = sample_noise_input(wl.grid, 0, spec.in_channels, 0.1)
    threads = os.cpu_count()
    torch.set_num_threads(threads)
    r = OracleFrameOptimizer(spec.channels, spec.in_channels, noise.values, wl.matrix.values,
                             wl.matrix.columns_q(), wl.output_map, spec.learning_rate)
    kaiming_reset(r.model, 1)
    dv = wl.voltages.frames[0].values
    for _ in range(args.warmup):
        r.optimize(dv, [], 1, 1)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        r.optimize(dv, [], 1, 1)
    t = time.perf_counter() - t0
    v = args.steps / t
    out = {"metric": "DIP iters/sec", "value": round(v, 4), "unit": "it/s", "n_gpus": ws, "steps": args.steps,
           "warmup": args.warmup, "ms_per_step": round(1e3 * t / args.steps, 3), "higher_is_better": True,
           "scaling": "weak", "vs_baseline": None, "dtype": "f32", "impl": "reference",
           "data": "synthetic (seeded BASELINE cfg generator)",
           "config": {"workload": args.workload + ("" if args.net == "config" else
                                                f"+FastResUNet3D(b={args.base_channels},{'dense' if args.dense else 'depthwise'})"),
                   "grid": list(spec.grid), "channels": list(spec.channels),
                      "C_z": spec.in_channels, "M": int(wl.matrix.n_measurements), "V": int(wl.matrix.n_masked),
                      "parallelism": "CPU, rank 0 only"},
           "cpu_baseline": {"value": round(v, 4), "unit": "it/s", "cores": threads, "kind": "port",
                            "sample": f"{args.steps} DIP iterations of {args.workload} after {args.warmup} warm-up"},
           "e2e": {"value": round(v, 4), "unit": "it/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=300)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--workload", default="cfg1")
    ap.add_argument("--precision", default=None)
    ap.add_argument("--net", default="config", choices=["config", "fast"],
                    help="config: the BASELINE config ResUNet; fast: the reference's FastResUNet3D (NetworkConfig)")
    ap.add_argument("--base-channels", type=int, default=8)
    ap.add_argument("--dense", action="store_true", help="FastResUNet3D with dense 3^3 convs (use_depthwise=False)")
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--skip-e2e", action="store_true")
    ap.add_argument("--skip-cpu", action="store_true")
    ap.add_argument("--skip-probe", action="store_true", help="skip the 1.6 GB HBM probe of the J kernel")
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    ap.add_argument("--e2e-frames", type=int, default=20)
    ap.add_argument("--e2e-warm", type=int, default=2000)
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_gpu(args)


if __name__ == "__main__":
    main()
