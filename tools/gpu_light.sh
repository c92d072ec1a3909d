# light-budget sweep (exact mode hand-off to the warp-parallel search) (dev tool)
for ls in "$@"; do echo "== light $ls"; MPLD_LIGHT_STEPS=$ls timeout 300 python tools/kernel_times.py --replicas 16 --single 2>&1 | grep -v "^  rounds\|slowest disc" | tail -4; done
