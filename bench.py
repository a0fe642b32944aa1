"""Benchmark of the DIP step (BASELINE.json metric "DIP iters/sec & tsEIT frames/sec").

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload cfg1] [--impl reference]

A step is one DIP iteration (ResUNet forward + masked J.sigma data term +
adjoint + backward + Adam) of the workload, replayed from a CUDA graph with
every input resident in HBM. N=1 runs the largest single-GPU BASELINE config,
cfg2 (64x64x32 grid, 16/32/64/128 ResUNet, M=3,904, V=103,296: a 1.6 GB J,
TF32-class convolutions). The single-sequence workloads do not shard (the TPP
chain is sequential), so N>1 runs N independent replicas (one
sequence per rank, weak scaling) and `value` is the total iterations of all
ranks / the max over ranks of the device time. `--gpus N` without torchrun
re-launches itself under `torch.distributed.run` with N ranks.

`e2e` is the same metric through the public API: one `reconstruct_sequence`
call on host (numpy) inputs at the workload's budgets (cfg2: UPWS 1,000 +
100 frames x 50), host->device uploads of J / Z / dv and device->host reads of
traces, checksums and volumes inside the timed region.

`cpu_baseline` and `--impl reference` time the reference algorithm's CPU
implementation (the oracle port, `oracle/`, bit-exact to the reference
package on the golden cases) on the box's host cores: exactly one training
iteration (pipeline.py:310-331) per step against a persistent Adam, all host
threads (`cpu_baseline_serial`: 1 thread, the reference's `serial=True`).
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
    """nvidia-smi sampling (50 ms) from before the warm-up to the end of the timed
    region; `summary()` keeps the samples inside the marked timed window (all samples
    from the warm-up on when the window is shorter than the sampling period)."""

    Q = ("timestamp,index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.marks = {}
        self.path = Path(f"/tmp/d2ip_clocks_{os.getpid()}.csv")

    def __enter__(self):
        try:
            self.fh = open(self.path, "w")
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "50"],
                                         stdout=self.fh, stderr=subprocess.DEVNULL)
            time.sleep(0.3)  # let the sampler start before the warm-up
        except Exception:
            self.proc = None
        return self

    def mark(self, name):
        self.marks[name] = time.time()

    def __exit__(self, *a):
        if self.proc is not None:
            time.sleep(0.1)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
            self.fh.close()

    def summary(self):
        import datetime

        if self.proc is None or not self.path.exists():
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        rows = [r.split(", ") for r in self.path.read_text().strip().splitlines() if r.strip()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        samples = []
        for r in rows:
            try:
                ts = datetime.datetime.strptime(r[0].strip(), "%Y/%m/%d %H:%M:%S.%f").timestamp()
                samples.append((ts, float(r[2]), float(r[3]),
                                {n for n, v in zip(names, r[6:10]) if v.strip().lower() == "active"}))
            except (ValueError, IndexError):
                continue
        t0, t1 = self.marks.get("timed_start"), self.marks.get("timed_end")
        window = [x for x in samples if t0 is not None and t1 is not None and t0 - 0.05 <= x[0] <= t1 + 0.05]
        scope = "timed region"
        if len(window) < 3:
            window, scope = samples, "warm-up + timed region"
        if not window:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        mx = window[-1][2]
        sm = [x[1] for x in window]
        loaded = [v for v in sm if mx and v > 0.5 * mx] or sm
        reasons = sorted(set().union(*[x[3] for x in window]))
        return {"sm_mhz": statistics.median(loaded), "sm_max_mhz": mx, "reasons": reasons,
                "samples": len(window), "scope": scope}


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
    joint = None
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
    elif spec.joint_frames:
        # cfg4: the joint warm-start step -- one network over `joint_frames` frames, the
        # frames sharded over the ranks (n_rhs per rank), J (5.4 GB) synthesised on the GPU
        from paper_2507_14046_b200.distributed import shard
        mine = list(shard(spec.joint_frames, ws, rank))
        J_dev, mask, dvs, omap = W.device_frames(spec, 0, spec.joint_frames)
        wl = None
        net = spec.network(seed=1)
        grid = spec.geometry()
        noise = sample_noise_input(grid, 0, spec.in_channels, 0.1)
        dn = DeviceNet(net, grid.shape, J_dev.shape[0], mask, data_norm="l2sq", output_map=omap, n_rhs=len(mine),
                       lr=spec.learning_rate, precision=args.precision or spec.precision,
                       max_iters=args.warmup + args.steps + 8)
        dn.set_noise(noise.values)
        dn.set_J_device(J_dev)
        del J_dev
        dn.set_theta(kaiming_flat(net))
        dn.dv[0].copy_(dvs[mine])
        # the TPP phase's single-frame step on the same device J (rank 0)
        tpp = DeviceNet(net, grid.shape, dn.M, mask, data_norm="l2sq", output_map=omap, lr=spec.learning_rate,
                        precision=args.precision or spec.precision, max_iters=args.warmup + args.steps + 8)
        tpp.set_noise(noise.values)
        tpp.set_J(dn.J)
        tpp.set_theta(kaiming_flat(net))
        tpp.dv[0, 0].copy_(dvs[0])
        units_per_step = 1
        joint = {"frames": spec.joint_frames, "frames_this_rank": len(mine), "tpp_net": tpp}
    else:
        # cfg0-2: the seeded host workload (cfg2: 1.6 GB J, 100 frames), the same arrays
        # the e2e call and the CPU arm consume
        frames = spec.frames if not args.skip_e2e else 1
        wl = W.make_workload(spec, seed=seed, frames=frames)
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
    if joint is not None and ws > 1:
        from paper_2507_14046_b200.distributed import allreduce_grads, allreduce_status

        def step():  # grads graph -> NCCL all-reduce (grad SUM, status MAX) -> Adam
            dn.grads(graph=True)
            allreduce_grads(dn.grad)
            allreduce_status(dn.status)
            dn.adam()
    else:
        def step():
            dn.run(1)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    clk = Clocks(local).__enter__()  # sampler started before the warm-up so the timed region is covered
    try:
        for _ in range(args.warmup):
            step()
        torch.cuda.synchronize()
        if ws > 1:
            dist.barrier()
        torch.cuda.synchronize()
        clk.mark("timed_start")
        for i in range(args.steps):
            flush.zero_()  # L2 flush between timed iterations (outside the events)
            ev[i][0].record()
            step()
            ev[i][1].record()
        torch.cuda.synchronize()
        clk.mark("timed_end")
    finally:
        clk.__exit__()
    t_dev = sum(a.elapsed_time(b) for a, b in ev) / 1e3
    if ws > 1:
        t = torch.tensor([t_dev], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        t_dev = float(t.item())
        dist.barrier()
    status = dn.status_host()
    # (D2IP_BENCH_NOCHECK=1: timing studies with deliberately wrong kernels, e.g. D2IP_TC_DBG)
    assert status[0, 1] == 0 or os.environ.get("D2IP_BENCH_NOCHECK") == "1", "non-finite loss during the benchmark"
    launches = dn.launches_per_iter()
    # replicas / sharded sequences: every rank's units count; the joint warm-start is ONE
    # job split over the ranks (strong scaling): its iterations count once
    its = (1 if joint is not None else ws) * units_per_step * args.steps / t_dev

    # --- no-flush steady state (informational): J may stay L2-resident
    torch.cuda.synchronize()
    s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s0.record()
    for _ in range(args.steps):
        step()
    s1.record()
    torch.cuda.synchronize()
    its_hot = units_per_step * args.steps / (s0.elapsed_time(s1) / 1e3)
    tpp_its = None
    if joint is not None:  # the TPP phase (single frame, one GPU): graph-replayed steps, L2 flushed
        tn = joint.pop("tpp_net")
        tn.reset_frame()
        tn.run(args.warmup)
        tev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
        for i in range(args.steps):
            flush.zero_()
            tev[i][0].record()
            tn.run(1)
            tev[i][1].record()
        torch.cuda.synchronize()
        tpp_its = args.steps / (sum(a.elapsed_time(b) for a, b in tev) / 1e3)
        tn.close()

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
    if not args.skip_probe and dn.M * dn.Vp < 3904 * 103296:
        Vp2 = (103296 + 3) // 4 * 4
        J2 = torch.randn(3904, Vp2, device="cuda")
        hbm_probe = jac_probe(3904, Vp2, J2)
        del J2
    # dominant kernel: the tcgen05 conv on the workload's largest level-0 layer
    # (dec0.conv1, (c1 + c0) -> c0 channels at the full grid), one launch timed live
    conv_roof = None
    if args.net == "config" and spec.precision != "bf16":
        c0, c1 = spec.channels[0], spec.channels[1]
        conv_roof = conv_probe(L, N, C, st, pk, pk_kind, flush, t_flush, c0 + c1, c0, tuple(spec.grid),
                               args.workload)
    # the bf16 tensor-core kernels on cfg4's largest layer (dec0.conv1, 96 -> 32 at 96x96x48)
    conv_bf16 = None if args.skip_probe and spec.precision != "bf16" else conv_bf16_probe(L, N, C, st, flush, t_flush)
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
    if conv_roof is not None:
        roofline = conv_roof
    elif conv_bf16 is not None and spec.precision == "bf16":
        roofline = {"bound": "tensor", "kernel": conv_bf16["fwd"]["kernel"], "layer": conv_bf16["layer"],
                    "achieved": conv_bf16["fwd"]["achieved"], "peak": conv_bf16["peak"], "unit": "TFLOP/s",
                    "frac": conv_bf16["fwd"]["frac"], "traffic": conv_bf16.get("traffic"),
                    "algorithmic_flops_per_launch": conv_bf16["algorithmic_flops_per_launch"],
                    "avg_launch_s": conv_bf16["fwd"]["avg_launch_s"], "peak_source": conv_bf16["peak_source"]}
    else:
        roofline = jac_cfg

    # --- e2e through the public API (rank-local, one full sequence)
    e2e = None
    dims = (dn.M, dn.V)
    if not args.skip_e2e and joint is not None and ws == 1:
        dn.close()
        del dn
        torch.cuda.empty_cache()
        e2e = run_e2e_joint(spec, args)
    if not args.skip_e2e and spec.sequences > 1:
        e2e = run_e2e_batched(spec, args, ws, rank)
    if not args.skip_e2e and units_per_step == 1 and wl is not None and args.net == "config":
        e2e = run_e2e(spec, wl, args, ws)
        if ws > 1:  # replicas: all ranks' iterations over the slowest rank's wall time
            t = torch.tensor([e2e["seconds"], e2e["iterations"]], dtype=torch.float64, device="cuda")
            tt = t.clone()
            dist.all_reduce(t[:1], op=dist.ReduceOp.MAX)
            dist.all_reduce(tt[1:], op=dist.ReduceOp.SUM)
            e2e["value"] = round(float(tt[1]) / float(t[0]), 2)
            e2e["aggregate"] = f"sum of {ws} replicas' iterations / max seconds over ranks"

    out = {
        "metric": "DIP iters/sec", "value": round(its, 2), "unit": "it/s", "n_gpus": ws, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(1e3 * t_dev / args.steps, 4), "higher_is_better": True,
        "scaling": "strong" if joint is not None else "weak", "vs_baseline": None,
        "dtype": ("f32 (TF32-class convs: 3xbf16 hi/lo operand splits on kind::f16, fp32 accumulate)"
                  if os.environ.get("D2IP_TF32_BF3", "0") != "0" else "f32 (3xTF32 conv operands)")
                 if (args.precision or spec.precision) == "tf32" else
                 ("f32 (bf16 conv operands, fp32 accumulate; forwards on 3xbf16 hi/lo operands)"
                  if (args.precision or spec.precision) == "bf16" else "f32"),
        "data": "synthetic (seeded BASELINE cfg generator; random-init weights)",
        "config": {"workload": args.workload + ("" if args.net == "config" else
                                                f"+FastResUNet3D(b={args.base_channels},{'dense' if args.dense else 'depthwise'})"),
                   "grid": list(spec.grid), "channels": list(spec.channels),
                   "C_z": spec.in_channels, "M": dims[0], "V": dims[1], "n_params": units["n_params"],
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
        "data_setup": "host-generated seeded workload (J, 100 frames of dv), uploaded once before timing"
                      if wl is not None else "J and dv synthesised on the GPU (torch RNG, seeded)",
    }
    if joint is not None:
        out["metric"] = "DIP iters/sec (joint warm-start: one iteration = all joint frames)"
        out["config"]["joint_frames"] = joint["frames"]
        out["config"]["parallelism"] = (f"joint warm-start, {joint['frames']} frames sharded over {ws} GPU(s) "
                                        f"({joint['frames_this_rank']} per rank, NCCL all-reduce of the gradient)"
                                        if ws > 1 else f"joint warm-start, {joint['frames']} frames as right-hand sides")
        out["tpp_its_single_gpu"] = round(tpp_its, 2)
        out["frames_per_sec"] = round(spec.frames / (spec.iters_warm / its + spec.frames * spec.iters_next / tpp_its), 4)
    if units_per_step > 1:
        out["config"]["sequences_per_gpu"] = units_per_step
        out["config"]["parallelism"] = f"{spec.sequences} sequences sharded over {ws} GPU(s), batched in lockstep"
    if e2e is not None:
        out["e2e"] = e2e
    if rank == 0 and ws == 1 and not args.skip_cpu and args.net == "config" and wl is not None:
        out["cpu_baseline"] = cpu_baseline(spec, wl, seconds=args.cpu_seconds)
        out["cpu_baseline_serial"] = cpu_baseline(spec, wl, seconds=args.cpu_seconds, threads=1)
    if rank == 0:
        print(json.dumps(out))
    if ws > 1:
        dist.destroy_process_group()


# dense TF32 tensor peak measured with tools/umma_rate.cu (148 SMs x 2 CTAs,
# M=128 N=256 kind::tf32 MMAs): 1104.5 TFLOP/s (profiles/r1_umma_rate.txt)
TF32_PEAK_TFLOPS = 1104.5


def ncu_traffic(name):
    """DRAM read + write bytes of one launch from a committed `ncu --set full` summary."""
    try:
        prof = json.loads((ROOT / "profiles" / name).read_text())
        scale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
        return sum(float(prof[k]["value"].replace(",", "")) * scale[prof[k]["unit"]]
                   for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"))
    except Exception:
        return None


# committed ncu --set full captures of the probed conv layers (profiles/)
NCU_CONV = {"cfg1": "r1_ncu_cfg1dec0c1.json", "cfg2": "r2_ncu_cfg2dec0c1.json"}


def conv_probe(L, N, C, st, pk, pk_kind, flush, t_flush, cin=48, cout=16, dims=(32, 32, 32), workload="cfg1"):
    """One launch of the tcgen05 conv on the workload's dec0.conv1 shape ((c1 + c0) -> c0
    at the full grid; cfg2: 48 -> 16 @ 64x64x32), timed with CUDA events on the launch
    stream; algorithmic FLOPs = 2*27*Cin*Cout*V."""
    import torch

    Dd, Hd, Wd = dims
    V = Dd * Hd * Wd
    x = torch.randn(1, Dd, Hd, Wd, cin, device="cuda")
    y = torch.empty(1, Dd, Hd, Wd, cout, device="cuda")
    w = torch.randn(cout * cin * 27 + cout, device="cuda") * 0.05

    def act(t, c):
        a = N.Act()
        a.ptr, a.d, a.h, a.w, a.c, a.cstride = t.data_ptr(), Dd, Hd, Wd, c, c
        a.bstride = V * c
        return a

    wsn = L.d2ip_conv3d_ws_bytes(cin, cout, 3, 1, N.PREC["tf32"], 1)
    ws = torch.empty(wsn, dtype=torch.uint8, device="cuda")
    xa, ya = act(x, cin), act(y, cout)

    def run():
        flush.zero_()
        N.check(L.d2ip_conv3d_fwd(xa, C.c_void_p(w.data_ptr()), C.c_void_p(w.data_ptr() + 4 * cout * cin * 27), 0,
                                  3, 1, ya, 0, N.PREC["tf32"], C.c_void_p(ws.data_ptr()), wsn, 1, st), "conv")
    t = max(time_kernel(run) - t_flush, 1e-9)
    flops = 2.0 * 27 * cin * cout * V
    peak = pk.get("bf16_tflops", 1665.3)  # MEASURED_PEAKS.json: dense bf16 (the operand type the kernel runs)
    src = NCU_CONV.get(workload)
    traffic = ncu_traffic(src) if src else None
    b3 = os.environ.get("D2IP_TF32_BF3", "0") != "0"
    # shape bound: an M=128 x N=16 MMA reads 4 KB (A) + 0.5 KB (B) of shared memory in ~39 cycles
    # (tools/umma_chains.cu): kind::f16 does 2*128*16*16 flop in it (of 8,192 flop/cycle/SM at
    # the 2,209 TFLOP/s probe peak), kind::tf32 half that; 3x MMAs per fp32-accurate product
    f16_probe = F16_PEAK_TFLOPS
    n16 = f16_probe * (2 * 128 * 16 * 16 / 39) / 8192 / 3 if b3 else TF32_PEAK_TFLOPS * (2 * 128 * 16 * 8 / 39) / 4096 / 3
    del x, y, ws
    return {"bound": "tensor",
            "kernel": "conv_tc_k (K1, tcgen05 %s implicit GEMM) incl. weight pack" % ("3xbf16 kind::f16" if b3 else "3xTF32"),
            "layer": f"dec0.conv1 {cin}->{cout} @ {Dd}x{Hd}x{Wd}", "achieved": round(flops / t / 1e12, 2),
            "peak": peak, "unit": "TFLOP/s", "frac": round(flops / t / 1e12 / peak, 4), "traffic": traffic,
            "traffic_source": f"profiles/{src} (ncu --set full, dram read+write bytes)" if traffic else None,
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


def run_e2e_joint(spec, args):
    """cfg4 end to end through `reconstruct_sequence_joint` on host inputs: the joint warm
    start over `joint_frames` frames, then frame 1 + the TPP chain (bounded to
    --e2e-frames-joint frames), uploads / read-backs inside the timed region."""
    import torch

    from paper_2507_14046_b200 import reconstruct_sequence_joint
    from paper_2507_14046_b200 import workloads as W
    from paper_2507_14046_b200.forward import MaskedSensitivity, VoltageSequence

    frames = max(spec.joint_frames, min(spec.frames, args.e2e_frames_joint))
    wl = W.make_workload(spec, seed=0, frames=frames)
    cfg = W.run_config_for(spec, wl.output_map, seed=0, precision=args.precision or spec.precision)
    matrix = MaskedSensitivity(np.array(wl.matrix.values), wl.matrix.mask)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    res = reconstruct_sequence_joint(matrix, VoltageSequence(wl.voltages.frames), cfg, wl.grid,
                                     joint_frames=spec.joint_frames)
    torch.cuda.synchronize()
    secs = time.perf_counter() - t0
    iters = cfg.iters_warm + sum(f.iterations for f in res.frame_records)
    nparam = res.states["init"].flat().numel()
    h2d = matrix.values.nbytes + 4 * np.prod(wl.grid.shape) * spec.in_channels + (frames + spec.joint_frames) * 4 * \
        wl.matrix.n_measurements + 4 * nparam
    d2h = (frames + 1) * (4 * np.prod(wl.grid.shape) + 4 * nparam + 16) + 4 * iters * 4
    return {"value": round(iters / secs, 2), "unit": "it/s", "h2d_bytes_per_step": int(h2d / iters),
            "d2h_bytes_per_step": int(d2h / iters), "call": "reconstruct_sequence_joint",
            "iterations": int(iters), "frames": frames, "seconds": round(secs, 3),
            "frames_per_sec": round(frames / secs, 4),
            "note": f"joint warm-start ({cfg.iters_warm} iterations over {spec.joint_frames} frames) + frame 1 and "
                    f"a TPP chain of {frames - 1} frames ({cfg.iters_next} each): the 100-frame chain bounded to "
                    f"{frames} frames"}


def run_e2e_batched(spec, args, ws, rank):
    """cfg3 end to end through `reconstruct_sequences_batched` on host inputs: all the
    independent sequences (sharded over the ranks, one batched engine per rank, gathered on
    rank 0), bounded to --e2e-frames-batched frames and a --e2e-warm-batched warm start so the
    call stays short; uploads and read-backs inside the timed region. Time = max over ranks."""
    import torch
    import torch.distributed as dist

    from paper_2507_14046_b200 import reconstruct_sequences_batched
    from paper_2507_14046_b200 import workloads as W
    from paper_2507_14046_b200.distributed import shard

    frames = min(spec.frames, args.e2e_frames_batched)
    seeds = list(range(spec.sequences))
    mine = set(shard(len(seeds), ws, rank))
    wls = [W.make_workload(spec, seed=s, frames=frames) if s in mine else None for s in seeds]
    proto = next(w for w in wls if w is not None)
    # the non-local sequences are never touched on this rank: stand-ins with the same shapes
    mats = [w.matrix if w is not None else proto.matrix for w in wls]
    volts = [w.voltages if w is not None else proto.voltages for w in wls]
    cfg = W.run_config_for(spec, proto.output_map, seed=0, precision=args.precision or spec.precision,
                           iters_warm=min(spec.iters_warm, args.e2e_warm_batched))
    torch.cuda.synchronize()
    if ws > 1:
        dist.barrier()
    t0 = time.perf_counter()
    res = reconstruct_sequences_batched(mats, volts, cfg, proto.grid, seeds=seeds)
    torch.cuda.synchronize()
    secs = time.perf_counter() - t0
    if ws > 1:
        t = torch.tensor([secs], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        secs = float(t)
    per_seq = cfg.iters_warm + cfg.iters_first + (frames - 1) * cfg.iters_next
    iters = per_seq * len(seeds)
    Q = int(np.prod(proto.grid.shape))
    h2d = len(mine) * (proto.matrix.values.nbytes + 4 * Q * spec.in_channels + frames * 4 * proto.matrix.n_measurements)
    d2h = len(mine) * frames * 8 * Q
    return {"value": round(iters / secs, 2), "unit": "it/s", "h2d_bytes_per_step": int(h2d / (iters / ws)),
            "d2h_bytes_per_step": int(d2h / (iters / ws)), "call": "reconstruct_sequences_batched",
            "iterations": int(iters), "sequences": len(seeds), "frames": frames, "seconds": round(secs, 3),
            "note": f"{len(seeds)} sequences x (warm {cfg.iters_warm} + {frames} frames x {cfg.iters_next}); the "
                    f"50-frame, 2,000-iteration warm-start budget bounded for a short run"}


def _oracle_runner(spec, wl):
    from oracle import OracleFrameOptimizer
    from oracle.resunet import kaiming_reset
    from paper_2507_14046_b200.priornet import sample_noise_input

    noise = sample_noise_input(wl.grid, wl.seed, spec.in_channels, 0.1)
    r = OracleFrameOptimizer(spec.channels, spec.in_channels, noise.values, wl.matrix.values,
                             wl.matrix.columns_q(), wl.output_map, spec.learning_rate)
    kaiming_reset(r.model, wl.seed + 1)
    return r


def _time_iterations(r, dv, warmup, max_steps, budget_s):
    """Warm-up, then timed single training iterations (pipeline.py:310-331, persistent
    Adam) until `max_steps` or the time budget; returns (n, seconds)."""
    import torch

    dv_t = torch.as_tensor(np.asarray(dv), dtype=torch.float32)
    opt = r.iterate(dv_t, [], max(warmup, 1))
    n, t = 0, 0.0
    while n < max_steps and (t < budget_s or n < 2):
        t0 = time.perf_counter()
        r.iterate(dv_t, [], 1, opt)
        t += time.perf_counter() - t0
        n += 1
    return n, t


def cpu_baseline(spec, wl, seconds: float = 10.0, threads: int | None = None):
    """The oracle port (bit-exact to the reference on the golden cases) timed on the
    host cores on a bounded sample of the same workload: one training iteration per
    step, persistent Adam, no per-step output forward."""
    import torch

    threads = threads or os.cpu_count()
    prev = torch.get_num_threads()
    torch.set_num_threads(threads)
    try:
        r = _oracle_runner(spec, wl)
        n, t = _time_iterations(r, wl.voltages.frames[0].values, 1, 200, seconds)
    finally:
        torch.set_num_threads(prev)
    return {"value": round(n / t, 4), "unit": "it/s", "cores": threads, "kind": "port",
            "ms_per_iter": round(1e3 * t / n, 2),
            "sample": f"{n} DIP training iterations of {spec.name} after 1 warm-up (oracle port of "
                      f"pipeline.py:310-331, torch CPU fp32, {threads} thread(s), persistent Adam)",
            "cpu": _cpu_model()}


def _cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


def run_reference(args):
    ws, rank, local = dist_env()
    if rank != 0:
        return
    import torch

    from paper_2507_14046_b200 import workloads as W

    spec = W.CONFIGS[args.workload]
    if spec.n_measurements * int(np.prod(spec.grid)) > 512 * 1024 * 1024:
        print(json.dumps({"impl": "reference", "unavailable": f"{args.workload}: a 5.4 GB host J is outside "
                          "the CPU arm's bounded sample (use cfg0-cfg2)"}))
        return
    wl = W.make_workload(spec, seed=0, frames=1)
    threads = os.cpu_count()
    torch.set_num_threads(threads)
    r = _oracle_runner(spec, wl)
    # one training iteration per step; the run is bounded to ~90 s of timed CPU work
    n, t = _time_iterations(r, wl.voltages.frames[0].values, args.warmup, args.steps, args.ref_seconds)
    v = n / t
    out = {"metric": "DIP iters/sec", "value": round(v, 4), "unit": "it/s", "n_gpus": ws, "steps": n,
           "steps_requested": args.steps, "warmup": args.warmup, "ms_per_step": round(1e3 * t / n, 3),
           "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32", "impl": "reference",
           "data": "synthetic (seeded BASELINE cfg generator; random-init weights)",
           "config": {"workload": args.workload, "grid": list(spec.grid), "channels": list(spec.channels),
                      "C_z": spec.in_channels, "M": int(wl.matrix.n_measurements), "V": int(wl.matrix.n_masked),
                      "parallelism": "CPU, rank 0 only"},
           "cpu_baseline": {"value": round(v, 4), "unit": "it/s", "cores": threads, "kind": "port",
                            "sample": f"{n} DIP training iterations of {args.workload} after {args.warmup} warm-up "
                                      f"(one iteration per step, persistent Adam; capped at {args.ref_seconds:.0f} s)",
                            "cpu": _cpu_model()},
           "e2e": {"value": round(v, 4), "unit": "it/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out))


def relaunch_distributed(argv, n):
    """`--gpus N` without a torchrun environment: re-exec under torch.distributed.run."""
    import socket

    with socket.socket() as s_:
        s_.bind(("127.0.0.1", 0))
        port = s_.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", f"--master-port={port}", str(Path(__file__).resolve()), *argv]
    return subprocess.call(cmd)


def run_launch_selftest(args):
    """CPU check of the multi-rank launcher (gloo): every rank reports, rank 0 prints."""
    import torch
    import torch.distributed as dist

    ws, rank, _ = dist_env()
    dist.init_process_group("gloo")
    t = torch.tensor([float(rank + 1)])
    dist.all_reduce(t)
    if rank == 0:
        print(json.dumps({"launch_selftest": True, "world_size": ws, "rank_sum": float(t)}))
    dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--workload", default="cfg2")
    ap.add_argument("--precision", default=None)
    ap.add_argument("--net", default="config", choices=["config", "fast"],
                    help="config: the BASELINE config ResUNet; fast: the reference's FastResUNet3D (NetworkConfig)")
    ap.add_argument("--base-channels", type=int, default=8)
    ap.add_argument("--dense", action="store_true", help="FastResUNet3D with dense 3^3 convs (use_depthwise=False)")
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--skip-e2e", action="store_true")
    ap.add_argument("--skip-cpu", action="store_true")
    ap.add_argument("--skip-probe", action="store_true", help="skip the 1.6 GB HBM probe of the J kernel")
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    ap.add_argument("--ref-seconds", type=float, default=90.0, help="cap on the reference arm's timed CPU work")
    ap.add_argument("--e2e-frames", type=int, default=100)
    ap.add_argument("--e2e-warm", type=int, default=2000)
    ap.add_argument("--e2e-frames-joint", type=int, default=20)
    ap.add_argument("--e2e-frames-batched", type=int, default=3)
    ap.add_argument("--e2e-warm-batched", type=int, default=200)
    ap.add_argument("--launch-selftest", action="store_true", help=argparse.SUPPRESS)
    args = ap.parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(relaunch_distributed(sys.argv[1:], args.gpus))
    if args.launch_selftest:
        run_launch_selftest(args)
    elif args.impl == "reference":
        run_reference(args)
    else:
        run_gpu(args)


if __name__ == "__main__":
    main()
