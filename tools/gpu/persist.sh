D2IP_TC_PERSIST=1 timeout 600 python -m pytest tests/test_gpu_ops.py -q -x -k "conv" --timeout 500 2>&1 | grep -E "^E  |FAILED|passed|failed" | head -5
for a in "32 32 96x96x48 1" "96 32 96x96x48 1" "64 64 48x48x24 1" "16 16 64x64x32 1"; do for v in 0 1; do
  D2IP_TC_PERSIST=$v timeout 100 python tools/conv_bench.py $a 20 $( [ "$a" = "16 16 64x64x32 1" ] && echo tf32 || echo bf16) 2>&1 | grep -E "fwd|dgrad|rror" | sed "s/^/P=$v /"; done; done
for v in 0 1; do for w in cfg4 cfg2 cfg1; do D2IP_TC_PERSIST=$v timeout 300 python bench.py --workload $w --steps 20 --warmup 5 --skip-e2e --skip-cpu --skip-probe 2>/dev/null | python -c "import json,sys;d=json.load(sys.stdin);print('P=$v $w',d['value'])"; done; done
