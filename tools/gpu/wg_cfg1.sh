for a in "8 16 32 1" "16 16 32 1" "48 16 32 1" "32 32 16 1" "96 32 16 1" "64 64 8 1" "16 32 32 2" "32 64 16 2"; do
  timeout 100 python tools/conv_bench.py $a 50 tf32 2>&1 | grep wgrad
  D2IP_WGBF3_MIN=0 timeout 100 python tools/conv_bench.py $a 50 tf32 2>&1 | grep wgrad | sed 's/^/B3 /'
done
