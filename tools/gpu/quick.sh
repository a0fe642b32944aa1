timeout 800 python -m pytest tests -m gpu -q --timeout 600 2>&1 | grep -E '^E  |FAILED|passed|failed' | head -5
for w in cfg1 cfg2 cfg4; do timeout 300 python bench.py --workload $w --steps $([ $w = cfg1 ] && echo 300 || echo 20) --warmup 5 --skip-e2e --skip-cpu --skip-probe 2>/dev/null | python -c "import json,sys;d=json.load(sys.stdin);print('$w',d['value'])"; done
