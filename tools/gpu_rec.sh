# recovery A/B (dev tool): parity tests with a 10-minute cap, kernel times of default and variants
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
echo "== default"; timeout 120 python tools/kernel_times.py --replicas 16 --single 2>&1 | grep -v "rounds/lev\|slowest disc\|seeds" | tail -3
for v in "$@"; do echo "== $v"; MPLD_LIB=paper_2303_14335_b200/lib/variants/libmpld_$v.so timeout 120 python tools/kernel_times.py --replicas 16 --single 2>&1 | grep -v "rounds/lev\|slowest disc\|seeds" | tail -3; done
