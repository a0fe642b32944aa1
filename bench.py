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
                                          "--format=csv,noheader,nounits", "-lms", "200"],
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
    wl = W.make_workload(spec, seed=seed, frames=min(spec.frames, 20))
    net = spec.network(seed=seed + 1)
    noise = sample_noise_input(wl.grid, seed, spec.in_channels, 0.1)
    dn = DeviceNet(net, wl.grid.shape, wl.matrix.n_measurements, wl.matrix.mask, data_norm="l2sq",
                   output_map=wl.output_map, lr=spec.learning_rate, precision=args.precision or spec.precision,
                   max_iters=args.warmup + args.steps + 8)
    dn.set_noise(noise.values)
    dn.set_J_host(wl.matrix.values)
    dn.set_theta(kaiming_flat(net))
    dn.set_dv(wl.voltages.frames[0].values)
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
    its = ws * args.steps / t_dev

    # --- no-flush steady state (informational): J may stay L2-resident
    torch.cuda.synchronize()
    s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s0.record()
    dn.run(args.steps)
    s1.record()
    torch.cuda.synchronize()
    its_hot = args.steps / (s0.elapsed_time(s1) / 1e3)

    # --- roofline of the dominant kernels, timed live on this stream
    pk, pk_kind = peaks()
    units = algorithmic_units(spec, net, dn.M, dn.Vp)
    L = N.lib()
    st = C.c_void_p(torch.cuda.current_stream().cuda_stream)
    nseg = L.d2ip_jac_nseg(dn.Vp)
    part = torch.empty(dn.M * nseg, device="cuda")
    sig = torch.randn(dn.Vp, device="cuda")

    def jac_fwd():
        flush.zero_()
        N.check(L.d2ip_jac_fwd(C.c_void_p(dn.J.data_ptr()), 0, C.c_void_p(sig.data_ptr()), 0, dn.M, dn.Vp,
                               C.c_void_p(part.data_ptr()), nseg, 1, st), "jac_fwd")

    t_flush = time_kernel(lambda: flush.zero_())
    t_jac = max(time_kernel(jac_fwd) - t_flush, 1e-9)
    jac_gbs = units["jac_bytes_per_pass"] / t_jac / 1e9
    # whole-iteration tensor-throughput view of the convolutions
    conv_tflops = units["conv_flops"] / (t_dev / args.steps) / 1e12
    roofline = {"bound": "hbm", "kernel": "jac_fwd (K5, J.sigma GEMV)", "achieved": round(jac_gbs, 1),
                "peak": pk["hbm_gbs"], "unit": "GB/s", "frac": round(jac_gbs / pk["hbm_gbs"], 4),
                "traffic": None, "peak_source": pk_kind,
                "algorithmic_bytes_per_launch": units["jac_bytes_per_pass"],
                "avg_launch_s": t_jac}

    # --- e2e through the public API (rank-local, one full sequence)
    e2e = None
    if not args.skip_e2e:
        e2e = run_e2e(spec, wl, args, ws)

    out = {
        "metric": "DIP iters/sec", "value": round(its, 2), "unit": "it/s", "n_gpus": ws, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(1e3 * t_dev / args.steps, 4), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f32 (TF32 conv operands)" if (args.precision or spec.precision) == "tf32" else "f32",
        "data": "synthetic (seeded BASELINE cfg generator; random-init weights)",
        "config": {"workload": args.workload, "grid": list(spec.grid), "channels": list(spec.channels),
                   "C_z": spec.in_channels, "M": dn.M, "V": dn.V, "n_params": units["n_params"],
                   "precision": args.precision or spec.precision,
                   "parallelism": f"replicas x{ws}" if ws > 1 else "single GPU",
                   "l2": "flushed between timed iterations (256 MB write)"},
        "frames_per_sec": round(its / ws * spec.frames / (spec.iters_warm + spec.frames * spec.iters_next), 4),
        "its_no_flush": round(its_hot, 2),
        "conv_tflops_effective": round(conv_tflops, 3),
        "gpu_launches": launches * args.steps,
        "launches_per_step": launches,
        "roofline": roofline,
        "clocks": clk.summary(),
    }
    if e2e is not None:
        out["e2e"] = e2e
    if rank == 0 and ws == 1 and not args.skip_cpu:
        out["cpu_baseline"] = cpu_baseline(args.workload, seconds=args.cpu_seconds)
    if rank == 0:
        print(json.dumps(out))
    if ws > 1:
        dist.destroy_process_group()


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
    h2d += 4 * nparam * (frames + 1)  # theta upload per stage
    d2h = frames * (8 * np.prod(wl.grid.shape) + 4 * nparam) + 4 * iters * 4
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
           "config": {"workload": args.workload, "grid": list(spec.grid), "channels": list(spec.channels),
                      "C_z": spec.in_channels, "M": int(wl.matrix.n_measurements), "V": int(wl.matrix.n_masked),
                      "parallelism": "CPU, rank 0 only"},
           "cpu_baseline": {"value": round(v, 4), "unit": "it/s", "cores": threads, "kind": "port",
                            "sample": f"{args.steps} DIP iterations of {args.workload} after {args.warmup} warm-up"},
           "e2e": {"value": round(v, 4), "unit": "it/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--workload", default="cfg1")
    ap.add_argument("--precision", default=None)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--skip-e2e", action="store_true")
    ap.add_argument("--skip-cpu", action="store_true")
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
