python -c 'import __graft_entry__ as g; g.smoke()' > gpurun_out/smoke.log 2>&1; tail -1 gpurun_out/smoke.log
timeout 900 python -m pytest tests -m gpu -q --timeout 800 2>&1 | tail -1
timeout 600 python bench.py > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err
timeout 400 python bench.py --workload cfg4 --steps 20 --warmup 5 --skip-e2e --skip-cpu --skip-probe > gpurun_out/bench_cfg4.json 2>/dev/null
bash tools/gpu/launches.sh cfg1 cfg1 > /dev/null 2>&1
