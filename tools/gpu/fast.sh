timeout 900 python -m pytest tests/test_gpu_refnet.py -m gpu -q 2>&1 | tail -1
for r in 1 2; do timeout 300 python bench.py --net fast --steps 200 --warmup 5 --skip-e2e --skip-cpu --skip-probe 2>/dev/null | python -c "import json,sys;d=json.load(sys.stdin);print('fast cfg1',d['value'])"; done
