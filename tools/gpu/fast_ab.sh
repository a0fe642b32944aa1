# A/B of two prebuilt libraries (ab_old.so / ab_new.so) on the FastResUNet3D bench
for r in 1 2; do for v in old new; do cp ab_$v.so paper_2507_14046_b200/_d2ip_b200.so
timeout 300 python bench.py --net fast --steps 200 --warmup 5 --skip-e2e --skip-cpu --skip-probe 2>/dev/null | python -c "import json,sys;d=json.load(sys.stdin);print('$v fast cfg1',d['value'])"; done; done
