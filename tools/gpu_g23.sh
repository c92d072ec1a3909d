timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout 120 python tools/kernel_times.py --replicas 16 --single 2>&1 | grep us_per | cut -c1-330
timeout 300 python bench.py --config 2 --steps 3 --no-cpu-baseline 2>&1 | tail -1 | cut -c1-250
python - <<'PY'
import json
d=json.loads(open('/dev/stdin').read()) if False else None
PY
