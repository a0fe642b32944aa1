run() { env "$@" timeout 300 python bench.py --steps 300 --warmup 5 --skip-e2e --skip-cpu --skip-probe 2>/dev/null | python -c "import json,sys;d=json.load(sys.stdin);print('$*',d['value'])"; }
run D2IP_X=0
run D2IP_WG_CTAS=296
run D2IP_WG_CTAS=444
run D2IP_WG_CTAS=222
