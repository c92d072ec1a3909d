# round 2: wide lane kernel check + configs[2]/[4] breakdown (dev tool)
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q -x -k "stress or exact or config2 or k4 or spill or edge or random or capacity" > gpurun_out/t_r2b.log 2>&1; tail -5 gpurun_out/t_r2b.log
for c in 2 4; do timeout 900 python bench.py --config $c --steps 5 --warmup 2 --no-cpu-baseline > gpurun_out/b_r2b_c$c.json 2> gpurun_out/b_r2b_c$c.err; tail -3 gpurun_out/b_r2b_c$c.err; python -c "
import json; d=json.load(open('gpurun_out/b_r2b_c$c.json')); print($c, d['ms_per_step'], d['value'], json.dumps(d['kernel_share']), json.dumps(d['stats'])); print(json.dumps(d.get('per_size')))"; done
