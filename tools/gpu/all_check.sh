timeout 900 python -m pytest tests -m gpu -q -x --timeout 600 2>&1 | grep -E "^E  |FAILED|passed|failed" | head -8
timeout 300 python bench.py --steps 100 --warmup 5 --skip-e2e --skip-cpu --skip-probe 2>/dev/null | head -c 120; echo
for w in cfg2 cfg4; do timeout 300 python bench.py --workload $w --steps 10 --warmup 3 --skip-e2e --skip-cpu --skip-probe 2>/dev/null | head -c 120; echo; done
