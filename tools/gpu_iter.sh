# parity tests + per-kernel times of the default build and the variants given as arguments (dev tool)
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
echo "== default"; timeout 300 python tools/kernel_times.py --replicas 16 --single 2>&1 | tail -6
for v in "$@"; do echo "== $v"; MPLD_LIB=paper_2303_14335_b200/lib/variants/libmpld_$v.so timeout 300 python tools/kernel_times.py --replicas 16 --single 2>&1 | tail -6; done
