# e2e A/B: round-1 snapshot vs current (dev tool)
mkdir -p gpurun_out
for i in 1 2; do
(cd r1snap && timeout 300 python bench.py --steps 10 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('r1', d['ms_per_step'], d['e2e']['ms_per_step'])")
timeout 300 python bench.py --steps 10 --no-cpu-baseline --no-secondary 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('r2', d['ms_per_step'], d['e2e']['ms_per_step'])"
done
timeout 300 python tools/e2e_probe.py
