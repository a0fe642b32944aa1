timeout 900 python -m pytest tests -m gpu -q -x --timeout 600 2>&1 | tail -3
for w in cfg2 cfg4; do timeout 400 python bench.py --workload $w --steps 10 --warmup 3 --skip-e2e --skip-cpu > gpurun_out/bench_$w.json 2> gpurun_out/bench_$w.err; head -c 250 gpurun_out/bench_$w.json; echo; done
timeout 300 python tools/trace_step.py --workload cfg4 --reps 1 --out gpurun_out/trace_cfg4.txt > /dev/null 2>&1; tail -4 gpurun_out/trace_cfg4.txt
