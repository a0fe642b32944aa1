timeout 900 python -m pytest tests/test_gpu_ops.py -q -x -k conv --timeout 600 2>&1 | grep -E "passed|failed|Error|assert" | head -5
for a in "32 32 96x96x48 1" "96 32 96x96x48 1" "64 64 48x48x24 1" "192 64 48x48x24 1" "8 32 96x96x48 1"; do
  timeout 120 python tools/conv_bench.py $a 20 bf16 2>&1 | grep -E "bf16"
done
