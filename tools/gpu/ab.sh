# usage: bash tools/gpu/ab.sh ENVVAR   -- cfg1 / cfg2 bench with ENVVAR=1 vs 0
for v in 1 0; do for w in cfg1 cfg2; do
 env $1=$v timeout 300 python bench.py --workload $w --steps $([ $w = cfg1 ] && echo 200 || echo 20) --warmup 5 --skip-e2e --skip-cpu --skip-probe 2>/dev/null | python -c "import json,sys;d=json.load(sys.stdin);print('$1=$v','$w',d['value'])"
done; done
