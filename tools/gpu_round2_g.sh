# round 2: exact mode hands > 32-vertex components to the heavy search unsearched (dev tool)
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -x > gpurun_out/t_r2g.log 2>&1; tail -3 gpurun_out/t_r2g.log
for i in 1 2; do timeout 900 python bench.py --config 2 --steps 5 --warmup 2 --no-cpu-baseline > gpurun_out/b_r2g_c2.json 2> gpurun_out/b_r2g_c2.err; tail -3 gpurun_out/b_r2g_c2.err; python -c "
import json; d=json.load(open('gpurun_out/b_r2g_c2.json')); print(2, d['ms_per_step'], d['value'], json.dumps(d['kernel_share']), json.dumps(d['stats']))"; done
for i in 1 2; do timeout 300 python bench.py --steps 10 --no-cpu-baseline --no-secondary 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c1', d['ms_per_step'], d['e2e']['ms_per_step'], json.dumps(d['kernel_share']))"; done
