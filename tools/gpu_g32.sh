timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "sharded or spill" 2>&1 | tail -2
for r in 1 2; do for v in default prespill; do L=""; [ $v != default ] && L=paper_2303_14335_b200/lib/variants/libmpld_$v.so; echo "== $v"; MPLD_LIB=$L timeout 120 python tools/kernel_times.py --replicas 16 --single 2>&1 | grep us_per | cut -c60-250; done; done
