#!/bin/bash
# Build locally, then run the GPU test suite + a short bench + launch list on a B200 box.
# usage: ./gpu_check.sh <tag> [extra command]
set -e
cd /root/repo
python build_ext.py > /tmp/build.log 2>&1 || { grep -i error /tmp/build.log | head; exit 1; }
TAG=${1:-x}
timeout 2400 /usr/local/graft/bin/gpurun --timeout 1500 -- "timeout 900 python -m pytest tests -m gpu -q --timeout 800 2>&1 | grep -E '^E  |passed|failed|FAILED' | head -14; timeout 300 python bench.py --steps 30 --warmup 5 --skip-cpu --skip-e2e > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; head -c 200 gpurun_out/bench_$TAG.json; echo; python bench.py --steps 1 --warmup 3 --skip-e2e --skip-cpu > gpurun_out/plain.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 1 --warmup 3 --skip-e2e --skip-cpu > gpurun_out/ncu.log 2>&1; echo ncu \$?; $2" 2>&1 | grep -v "^\[gpurun\] sending" | tail -20
