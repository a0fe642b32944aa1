"""bench.py contract pieces that run without a GPU: the `--gpus N` self-launch under
torch.distributed.run (gloo, world size 2) and the reference arm's JSON line (one
training iteration per step of the oracle port, rank 0 only)."""

import json
import subprocess
import sys

from conftest import ROOT


def _json_lines(out: str):
    return [json.loads(l) for l in out.splitlines() if l.startswith("{")]


def test_gpus_flag_relaunches_world_size_2():
    res = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--gpus", "2", "--launch-selftest"],
                         capture_output=True, text=True, timeout=300, cwd=ROOT)
    assert res.returncode == 0, res.stderr[-2000:]
    lines = _json_lines(res.stdout)
    assert lines == [{"launch_selftest": True, "world_size": 2, "rank_sum": 3.0}]


def test_reference_arm_line_under_two_ranks():
    res = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--impl", "reference", "--gpus", "2",
                          "--workload", "cfg0", "--steps", "3", "--warmup", "1"],
                         capture_output=True, text=True, timeout=300, cwd=ROOT)
    assert res.returncode == 0, res.stderr[-2000:]
    (line,) = _json_lines(res.stdout)  # rank 0 alone prints
    assert line["impl"] == "reference" and line["steps"] == 3 and line["n_gpus"] == 2
    assert line["metric"] == "DIP iters/sec" and line["unit"] == "it/s" and line["higher_is_better"]
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["cpu_baseline"]["kind"] == "port"
    assert abs(line["ms_per_step"] * line["value"] - 1e3) < 1e-3 * 1e3
