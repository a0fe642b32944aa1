for a in "32 32 96x96x48 1" "96 32 96x96x48 1"; do for v in 0 1; do D2IP_TC_DBG=$v timeout 100 python tools/conv_bench.py $a 20 bf16 | grep -E "fwd" | sed "s/^/DBG=$v /"; done; done
