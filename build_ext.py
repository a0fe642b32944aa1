"""Build the sm_100a extension in-tree: paper_2507_14046_b200/_d2ip_b200.so.

    python build_ext.py            # incremental (objects under build/)
    python build_ext.py --force

nvcc -gencode arch=compute_100a,code=sm_100a -lineinfo -O3, static cudart,
one shared object exporting the C ABI of include/d2ip_b200.h.
"""

from __future__ import annotations

import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

ROOT = Path(__file__).resolve().parent
CSRC = ROOT / "paper_2507_14046_b200" / "csrc"
OUT = ROOT / "paper_2507_14046_b200" / "_d2ip_b200.so"
BUILD = ROOT / "build" / "obj"
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "--expt-relaxed-constexpr",
         "-Xptxas", "-v,-warn-spills", "-I", str(ROOT / "include")]


def sources():
    return sorted(CSRC.glob("*.cu"))


def headers():
    return sorted(CSRC.glob("*.cuh")) + sorted(CSRC.glob("*.h")) + [ROOT / "include" / "d2ip_b200.h"]


def build(force: bool = False, verbose: bool = False) -> Path:
    BUILD.mkdir(parents=True, exist_ok=True)
    hdr_mtime = max(p.stat().st_mtime for p in headers())
    objs, todo = [], []
    for src in sources():
        obj = BUILD / (src.stem + ".o")
        objs.append(obj)
        if not force and obj.exists() and obj.stat().st_mtime > max(src.stat().st_mtime, hdr_mtime):
            continue
        todo.append((src, obj))

    def compile_one(job):
        src, obj = job
        cmd = [NVCC, *ARCH, *FLAGS, "-c", str(src), "-o", str(obj)]
        return src, obj, subprocess.run(cmd, capture_output=True, text=True)

    # translation units compile independently: in parallel, the largest first
    todo.sort(key=lambda j: -j[0].stat().st_size)
    with ThreadPoolExecutor(max_workers=max(1, min(len(todo), os.cpu_count() or 1))) as pool:
        for src, obj, res in pool.map(compile_one, todo):
            if res.returncode != 0:
                sys.stderr.write(res.stdout + res.stderr)
                raise RuntimeError(f"nvcc failed on {src.name}")
            (BUILD / (src.stem + ".ptxas.log")).write_text(res.stdout + res.stderr)
            if verbose:
                print(res.stderr)
    if force or not OUT.exists() or OUT.stat().st_mtime < max(o.stat().st_mtime for o in objs):
        cmd = [NVCC, *ARCH, "-shared", "-cudart", "static", "-o", str(OUT), *map(str, objs), "-lcuda"]
        res = subprocess.run(cmd, capture_output=True, text=True)
        if res.returncode != 0:
            sys.stderr.write(res.stdout + res.stderr)
            raise RuntimeError("link failed")
    return OUT


if __name__ == "__main__":
    p = build(force="--force" in sys.argv, verbose="-v" in sys.argv)
    print(p)
