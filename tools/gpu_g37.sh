timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
timeout 120 python tools/kernel_times.py --replicas 16 --single 2>&1 | grep us_per | cut -c60-300
for i in 1 2; do timeout 300 python bench.py --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],4))"; done
