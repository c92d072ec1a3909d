# round 2: compact heavy frames + staged light search (dev tool)
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -x > gpurun_out/t_r2d.log 2>&1; tail -3 gpurun_out/t_r2d.log
for c in 2 4; do timeout 900 python bench.py --config $c --steps 5 --warmup 2 --no-cpu-baseline > gpurun_out/b_r2d_c$c.json 2> gpurun_out/b_r2d_c$c.err; tail -3 gpurun_out/b_r2d_c$c.err; python -c "
import json; d=json.load(open('gpurun_out/b_r2d_c$c.json')); print($c, d['ms_per_step'], d['value'], json.dumps(d['kernel_share']), json.dumps(d['stats'])); print(json.dumps(d.get('per_size')))"; done
for i in 1 2; do timeout 300 python bench.py --steps 10 --no-cpu-baseline --no-secondary 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c1', d['ms_per_step'], d['e2e']['ms_per_step'], json.dumps(d['kernel_share']))"; done
timeout 300 python tools/kernel_times.py 2>&1 | tail -12
