timeout 600 python -m pytest tests/test_gpu_ops.py -q -x -k "dgrad_wgrad and bf16" --timeout 500 2>&1 | tail -1
D2IP_WB_SINGLE=1 timeout 600 python -m pytest tests/test_gpu_ops.py -q -x -k "dgrad_wgrad and bf16" --timeout 500 2>&1 | tail -1
for v in 0 1; do for a in "32 32 96x96x48 1" "96 32 96x96x48 1"; do D2IP_WB_SINGLE=$v timeout 100 python tools/conv_bench.py $a 20 bf16 | grep wgrad | sed "s/^/S=$v /"; done; done
for v in 0 1; do D2IP_WB_SINGLE=$v timeout 300 python bench.py --workload cfg4 --steps 20 --warmup 5 --skip-e2e --skip-cpu --skip-probe 2>/dev/null | python -c "import json,sys;d=json.load(sys.stdin);print('S=$v cfg4',d['value'])"; done
