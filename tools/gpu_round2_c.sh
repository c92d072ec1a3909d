# round 2: seeded incumbent check (dev tool)
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q -x -k "exact or config2 or k4 or spill or random or config1 or bench_launch" > gpurun_out/t_r2c.log 2>&1; tail -3 gpurun_out/t_r2c.log
for c in 2; do timeout 900 python bench.py --config $c --steps 5 --warmup 2 --no-cpu-baseline > gpurun_out/b_r2c_c$c.json 2> gpurun_out/b_r2c_c$c.err; tail -3 gpurun_out/b_r2c_c$c.err; python -c "
import json; d=json.load(open('gpurun_out/b_r2c_c$c.json')); print($c, d['ms_per_step'], d['value'], json.dumps(d['kernel_share']), json.dumps(d['stats']))"; done
timeout 300 python bench.py --steps 10 --no-cpu-baseline --no-secondary 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c1', d['ms_per_step'], d['e2e']['ms_per_step'], json.dumps(d['kernel_share']))"
