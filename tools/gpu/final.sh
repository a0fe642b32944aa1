python -c 'import __graft_entry__ as g; g.smoke()' > gpurun_out/smoke.log 2>&1; tail -1 gpurun_out/smoke.log
timeout 600 python bench.py > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err
for w in cfg2 cfg3 cfg4; do timeout 400 python bench.py --workload $w --steps 20 --warmup 5 --skip-e2e --skip-cpu --skip-probe > gpurun_out/bench_$w.json 2>/dev/null; done
bash tools/gpu/launches.sh cfg1 cfg1 > /dev/null 2>&1
bash tools/gpu/launches.sh cfg4 cfg4 > /dev/null 2>&1
python tools/conv_bench.py 96 32 96x96x48 1 3 bf16 > /dev/null 2>&1 && KREGEX=conv_tcp_k bash tools/gpu/ncu_conv.sh cfg4dec0c1 '96 32 96x96x48 1' bf16 > /dev/null 2>&1
KREGEX=wgrad_bf_k bash tools/gpu/ncu_conv.sh cfg4dec0c1wg '96 32 96x96x48 1' bf16 > /dev/null 2>&1
python tools/conv_bench.py 48 16 32 1 3 tf32 > /dev/null 2>&1 && KREGEX=conv_tc_k bash tools/gpu/ncu_conv.sh cfg1dec0c1 '48 16 32 1' tf32 > /dev/null 2>&1
ls gpurun_out/ncu_cfg*raw.csv
