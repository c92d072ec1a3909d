# round 2: full GPU suite, smoke, default bench line, launch lists and ncu --set full of configs[1]
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -x --durations=10 > gpurun_out/t_final.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/t_final.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_final.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke_final.log
timeout 900 python bench.py > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err; echo "bench rc=$?"
python -c "
import json; d=json.loads(open('gpurun_out/bench_final.json').read().strip().splitlines()[-1])
print('c1', d['value'], d['ms_per_step'], d['e2e']['value'], d['roofline']['kernel'], round(d['roofline']['frac'],4))
for k,v in d['secondary'].items():
    if k != 'configs[4]': print(k, v['value'], v['ms_per_step'])
"
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_final_c1.csv python bench.py --profile-launches --steps 2 --warmup 1 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:mpld_ -s 7 -c 7 -o gpurun_out/full_final_c1 -f python bench.py --profile-launches --steps 1 --warmup 1 > gpurun_out/ncu_final_c1.log 2>&1; tail -1 gpurun_out/ncu_final_c1.log
timeout 300 python bench.py --profile-launches --steps 1 --warmup 1 > gpurun_out/profile_run_final_c1.json 2>/dev/null
