export PYTORCH_NO_CUDA_MEMORY_CACHING=1
timeout 1200 /usr/local/cuda/bin/compute-sanitizer --tool memcheck --leak-check no --error-exitcode 9 --print-limit 20 \
  python -m pytest tests/test_gpu_ops.py -q -x --timeout 1100 -k "conv and (bf16 or tf32) and not 64-64-32 and not 48-48-32 and not 32-32-32 and not 65-34" 2>&1 | tail -25
echo "rc=$?"
timeout 900 /usr/local/cuda/bin/compute-sanitizer --tool memcheck --leak-check no --error-exitcode 9 --print-limit 20 \
  python -m pytest tests/test_gpu_engine.py -q -x --timeout 800 -k "three_level and mini" 2>&1 | tail -8
