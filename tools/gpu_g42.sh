timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for r in 1 2; do for v in default c8; do L=""; [ $v != default ] && L=paper_2303_14335_b200/lib/variants/libmpld_$v.so; MPLD_LIB=$L timeout 300 python bench.py --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', round(d['ms_per_step'],4))"; done; done
