python tools/conv_bench.py 48 16 32 1 3 tf32 > /dev/null 2>&1 && KREGEX=conv_tc_k bash tools/gpu/ncu_conv.sh cfg1dec0c1 '48 16 32 1' tf32
python -c 'import __graft_entry__ as g; g.smoke()' > gpurun_out/smoke.log 2>&1; tail -1 gpurun_out/smoke.log
timeout 600 python bench.py > gpurun_out/bench_s5.json 2> gpurun_out/bench_s5.err
bash tools/gpu/launches.sh cfg1 cfg1 > /dev/null 2>&1
bash tools/gpu/launches.sh cfg2 cfg2 > /dev/null 2>&1
