run() { env "$@" timeout 300 python bench.py --steps 300 --warmup 5 --skip-e2e --skip-cpu --skip-probe 2>/dev/null | python -c "import json,sys;d=json.load(sys.stdin);print('$*',d['value'])"; }
run D2IP_X=0
run D2IP_WG_SMEM_KB=100
run D2IP_WG_SMEM_KB=64
run D2IP_WG_CTAS=74
run D2IP_WG_CTAS=74 D2IP_WG_SMEM_KB=100
run D2IP_WG_CTAS=296 D2IP_WG_SMEM_KB=100
