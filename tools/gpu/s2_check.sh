for a in "16 32 32 2" "32 64 16 2" "8 16 32 1" "16 16 32 1" "48 16 32 1"; do
  timeout 100 python tools/conv_bench.py $a 50 tf32 2>&1 | grep -E "fwd|dgrad"
  D2IP_TC_S2=2 timeout 100 python tools/conv_bench.py $a 50 tf32 2>&1 | grep -E "fwd|dgrad" | sed 's/^/S2TC /'
done
