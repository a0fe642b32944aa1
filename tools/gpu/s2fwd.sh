# A/B: stride-2 3^3 forward convs on tcgen05 at every size (D2IP_TC_S2=2) vs the size rule (1)
python build_ext.py >/dev/null 2>&1 || { echo build failed; exit 1; }
for s in 1 2; do D2IP_TC_S2=$s timeout 120 python tools/conv_bench.py 16 32 32 2 200 tf32 2>&1 | sed "s/^/S2=$s 16->32 32^3: /"; done
for s in 1 2; do D2IP_TC_S2=$s timeout 120 python tools/conv_bench.py 32 64 16 2 200 tf32 2>&1 | sed "s/^/S2=$s 32->64 16^3: /"; done
for r in 1 2; do for s in 1 2; do for w in cfg1 cfg2; do
 D2IP_TC_S2=$s timeout 300 python bench.py --workload $w --steps $([ $w = cfg1 ] && echo 300 || echo 20) --warmup 5 --skip-e2e --skip-cpu --skip-probe 2>/dev/null | python -c "import json,sys;d=json.load(sys.stdin);print('S2=$s','$w',d['value'])"
done; done; done
