# per-kernel times of the default build and variants, twice (dev tool)
for r in 1 2; do for v in default "$@"; do L=""; [ $v != default ] && L=paper_2303_14335_b200/lib/variants/libmpld_$v.so; MPLD_LIB=$L timeout 120 python tools/kernel_times.py --replicas 16 --single 2>&1 | grep "us_per" | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', d['us_per_launch'])"; done; done
