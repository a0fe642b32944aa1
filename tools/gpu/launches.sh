# usage: bash tools/gpu/launches.sh TAG WORKLOAD [extra bench args]
TAG=$1; WL=$2; shift 2
timeout 400 python bench.py --workload $WL --steps 1 --warmup 3 --skip-e2e --skip-cpu --skip-probe "$@" > gpurun_out/plain_$TAG.log 2>&1 || { echo plain failed; tail -5 gpurun_out/plain_$TAG.log; exit 1; }
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 900 --csv --log-file gpurun_out/launches_$TAG.csv python bench.py --workload $WL --steps 1 --warmup 3 --skip-e2e --skip-cpu --skip-probe "$@" > gpurun_out/ncu_$TAG.log 2>&1
echo ncu rc $?
python profiles/summarize_launches.py gpurun_out/launches_$TAG.csv > gpurun_out/launches_$TAG.txt; head -30 gpurun_out/launches_$TAG.txt; tail -1 gpurun_out/launches_$TAG.txt
