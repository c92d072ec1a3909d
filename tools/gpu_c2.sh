timeout 900 python -m pytest tests -m gpu -x -q -k "spill or exact or qpld or k4 or stress" 2>&1 | tail -1
for i in 1 2; do timeout 300 python bench.py --config 2 --steps 5 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c2', round(d['ms_per_step'],3))"; done
timeout 300 python bench.py --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c1', round(d['ms_per_step'],4))"
