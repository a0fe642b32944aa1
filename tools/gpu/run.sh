#!/bin/bash
# GPU-box helper (run under gpurun from the repo root).  One script, sub-commands:
#
#   bash tools/gpu/run.sh tests [pytest -k expr]      GPU test suite (+ smoke)
#   bash tools/gpu/run.sh bench WL [STEPS] [args..]   one bench line  -> gpurun_out/bench_WL.json
#   bash tools/gpu/run.sh ab ENVVAR WL [WL..]         bench value with ENVVAR=1 vs ENVVAR=0
#   bash tools/gpu/run.sh launches TAG WL [args..]    ncu launch list (after a clean run) -> gpurun_out/launches_TAG.{csv,txt}
#   bash tools/gpu/run.sh ncu TAG KREGEX "cin cout dims stride" PREC
#                                                     ncu --set full of one conv kernel (tools/conv_bench.py)
#   bash tools/gpu/run.sh convs PREC "a" "b" ..      conv_bench over layer shapes
#   bash tools/gpu/run.sh sanitize [-k expr]          compute-sanitizer memcheck over the op tests
set -u
cmd=${1:-tests}; shift || true
steps_of() { case $1 in cfg1|cfg0) echo 300;; *) echo 20;; esac; }
value() { python -c "import json,sys;d=json.loads(sys.stdin.readline());print(d.get('value'), d.get('e2e',{}) and d['e2e'].get('value'))"; }
case $cmd in
tests)
  python -c 'import __graft_entry__ as g; g.smoke()' 2>&1 | tail -1
  timeout 1500 python -m pytest tests -m gpu -q --timeout 1200 ${1:+-k "$1"} 2>&1 | grep -E '^E  |FAILED|passed|failed|error' | head -20 ;;
bench)
  WL=$1; S=${2:-$(steps_of $1)}; shift; shift || true
  timeout 900 python bench.py --workload $WL --steps $S --warmup 5 "$@" > gpurun_out/bench_$WL.json 2> gpurun_out/bench_$WL.err
  echo "rc $?"; head -c 400 gpurun_out/bench_$WL.json; echo ;;
ab)
  V=$1; shift
  for w in "$@"; do for v in 1 0; do
    env $V=$v timeout 300 python bench.py --workload $w --steps $(steps_of $w) --warmup 5 --skip-e2e --skip-cpu --skip-probe 2>/dev/null | value | sed "s/^/$V=$v $w /"
  done; done ;;
launches)
  TAG=$1; WL=$2; shift 2
  timeout 400 python bench.py --workload $WL --steps 1 --warmup 3 --skip-e2e --skip-cpu --skip-probe "$@" > gpurun_out/plain_$TAG.log 2>&1 || { echo plain failed; tail -5 gpurun_out/plain_$TAG.log; exit 1; }
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 900 --csv --log-file gpurun_out/launches_$TAG.csv \
    python bench.py --workload $WL --steps 1 --warmup 3 --skip-e2e --skip-cpu --skip-probe "$@" > gpurun_out/ncu_$TAG.log 2>&1
  echo "ncu rc $?"
  python profiles/summarize_launches.py gpurun_out/launches_$TAG.csv > gpurun_out/launches_$TAG.txt
  head -25 gpurun_out/launches_$TAG.txt; tail -1 gpurun_out/launches_$TAG.txt ;;
ncu)
  TAG=$1; KR=$2; ARGS=$3; PREC=$4
  python tools/conv_bench.py $ARGS 3 $PREC > /dev/null 2>&1 || { echo "clean run failed"; exit 1; }
  timeout 400 ncu --set full --import-source on --clock-control none -k regex:$KR -c 1 -o gpurun_out/ncu_$TAG \
    python tools/conv_bench.py $ARGS 1 $PREC > gpurun_out/ncu_$TAG.log 2>&1
  echo "ncu rc $?"
  ncu -i gpurun_out/ncu_$TAG.ncu-rep --page details --csv > gpurun_out/ncu_$TAG.details.csv 2>/dev/null
  ncu -i gpurun_out/ncu_$TAG.ncu-rep --page raw --csv > gpurun_out/ncu_$TAG.raw.csv 2>/dev/null
  rm -f gpurun_out/ncu_$TAG.ncu-rep ;;
convs)
  PREC=$1; shift
  for a in "$@"; do timeout 120 python tools/conv_bench.py $a 20 $PREC 2>&1 | tail -4; done ;;
profiles)
  # round evidence: bench lines, launch lists, ncu --set full of the dominant kernels
  TAG=${1:-r2}
  timeout 900 python bench.py > gpurun_out/${TAG}_bench_cfg2.json 2> gpurun_out/${TAG}_bench_cfg2.err; echo "cfg2 rc $?"
  timeout 600 python bench.py --workload cfg1 --steps 300 > gpurun_out/${TAG}_bench_cfg1.json 2> gpurun_out/${TAG}_bench_cfg1.err; echo "cfg1 rc $?"
  timeout 600 python bench.py --workload cfg3 --steps 20 --skip-cpu > gpurun_out/${TAG}_bench_cfg3.json 2> gpurun_out/${TAG}_bench_cfg3.err; echo "cfg3 rc $?"
  timeout 900 python bench.py --workload cfg4 --steps 20 --skip-cpu > gpurun_out/${TAG}_bench_cfg4.json 2> gpurun_out/${TAG}_bench_cfg4.err; echo "cfg4 rc $?"
  for w in cfg2 cfg1 cfg4; do bash tools/gpu/run.sh launches ${TAG}_$w $w > /dev/null 2>&1; echo "launches $w $?"; done
  for spec in "cfg2dec0c1|conv_tc_k|48 16 64x64x32|fwd|tf32" "cfg2dec0c1dg|conv_tc_k|48 16 64x64x32|dgrad|tf32" \
              "cfg4dec0c1|conv_tc_k|96 32 96x96x48|fwd|bf16"; do
    IFS='|' read -r name kr shape dir prec <<< "$spec"
    python tools/conv_one.py $shape $dir 3 $prec > /dev/null 2>&1 || { echo "clean $name failed"; continue; }
    timeout 400 ncu --set full --import-source on --clock-control none -k regex:$kr -c 1 -o gpurun_out/ncu_$name \
      python tools/conv_one.py $shape $dir 1 $prec > gpurun_out/ncu_$name.log 2>&1
    ncu -i gpurun_out/ncu_$name.ncu-rep --page raw --csv > gpurun_out/ncu_$name.raw.csv 2>/dev/null
    python profiles/ncu_summary.py gpurun_out/ncu_$name.raw.csv gpurun_out/${TAG}_ncu_$name.json
    rm -f gpurun_out/ncu_$name.ncu-rep; echo "ncu $name done"
  done
  # the level-0 weight gradient (3xbf16, wgrad_bf_k) through conv_bench (fwd / dgrad / wgrad of one layer)
  name=cfg2dec0c1wg
  if python tools/conv_bench.py 48 16 64x64x32 1 3 tf32 > /dev/null 2>&1; then
    timeout 400 ncu --set full --import-source on --clock-control none -k regex:wgrad_bf_k -c 1 -o gpurun_out/ncu_$name \
      python tools/conv_bench.py 48 16 64x64x32 1 1 tf32 > gpurun_out/ncu_$name.log 2>&1
    ncu -i gpurun_out/ncu_$name.ncu-rep --page raw --csv > gpurun_out/ncu_$name.raw.csv 2>/dev/null
    python profiles/ncu_summary.py gpurun_out/ncu_$name.raw.csv gpurun_out/${TAG}_ncu_$name.json
    rm -f gpurun_out/ncu_$name.ncu-rep; echo "ncu $name done"
  fi ;;
sanitize)
  export PYTORCH_NO_CUDA_MEMORY_CACHING=1
  timeout 1200 /usr/local/cuda/bin/compute-sanitizer --tool memcheck --leak-check no --error-exitcode 9 --print-limit 20 \
    python -m pytest tests/test_gpu_ops.py -q -x --timeout 1100 "$@" 2>&1 | tail -25 ;;
*) echo "unknown sub-command $cmd"; exit 2 ;;
esac
