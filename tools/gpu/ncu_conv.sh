# usage: bash tools/gpu/ncu_conv.sh TAG "cin cout dims stride" prec
TAG=$1; ARGS=$2; PREC=$3
timeout 300 ncu --set full --import-source on --clock-control none -k regex:${KREGEX:-conv_tc_k} -c 1 -o gpurun_out/ncu_$TAG python tools/conv_bench.py $ARGS 1 $PREC > gpurun_out/ncu_$TAG.log 2>&1
echo ncu rc $?
ncu -i gpurun_out/ncu_$TAG.ncu-rep --page details --csv > gpurun_out/ncu_$TAG.details.csv 2>/dev/null
ncu -i gpurun_out/ncu_$TAG.ncu-rep --page raw --csv > gpurun_out/ncu_$TAG.raw.csv 2>/dev/null
ncu -i gpurun_out/ncu_$TAG.ncu-rep --page source --csv > gpurun_out/ncu_$TAG.source.csv 2>/dev/null
rm -f gpurun_out/ncu_$TAG.ncu-rep gpurun_out/ncu_$TAG.source.csv  # (keep the copy-back under 64 MiB)
ls -la gpurun_out/ncu_$TAG*
