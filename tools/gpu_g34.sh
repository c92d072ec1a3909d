timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
timeout 120 python tools/kernel_times.py --replicas 16 --single 2>&1 | grep us_per | cut -c60-300
timeout 300 python bench.py --config 2 --steps 3 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c2', round(d['ms_per_step'],2), d['stats']['steps'])"
