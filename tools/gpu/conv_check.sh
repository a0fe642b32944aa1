timeout 900 python -m pytest tests/test_gpu_ops.py -q -x -k conv --timeout 600 2>&1 | grep -E "passed|failed|Error|assert" | head -8
for a in "32 32 96x96x48 1" "96 32 96x96x48 1" "64 64 48x48x24 1" "192 64 48x48x24 1" "32 64 96x96x48 2" "128 128 24x24x12 1" "384 128 24x24x12 1" "8 32 96x96x48 1"; do timeout 120 python tools/conv_bench.py $a 20 ${PRECS:-tf32,bf16} 2>&1 | tail -6; done
