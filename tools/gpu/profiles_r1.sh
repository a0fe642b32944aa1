# ncu captures for profiles/ (each command first runs clean without ncu)
set -x
python tools/conv_bench.py 48 16 32 1 3 tf32 > /dev/null 2>&1 && KREGEX=conv_tc_k bash tools/gpu/ncu_conv.sh cfg1dec0c1 '48 16 32 1' tf32
python tools/conv_bench.py 96 32 96x96x48 1 3 bf16 > /dev/null 2>&1 && KREGEX=conv_tc_k bash tools/gpu/ncu_conv.sh cfg4dec0c1 '96 32 96x96x48 1' bf16
KREGEX=wgrad_bf_k bash tools/gpu/ncu_conv.sh cfg4dec0c1wg '96 32 96x96x48 1' bf16
bash tools/gpu/launches.sh cfg1 cfg1 > /dev/null 2>&1
bash tools/gpu/launches.sh cfg4 cfg4 > /dev/null 2>&1
ls gpurun_out/
