# round 2: ticketed ring claims, clique-term skip, staging syncwarp (dev tool)
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -x > gpurun_out/t_r2i.log 2>&1; tail -3 gpurun_out/t_r2i.log
for c in 2 4; do timeout 900 python bench.py --config $c --steps 5 --warmup 2 --no-cpu-baseline > gpurun_out/b_r2i_c$c.json 2> gpurun_out/b_r2i_c$c.err; tail -3 gpurun_out/b_r2i_c$c.err; python -c "
import json; d=json.load(open('gpurun_out/b_r2i_c$c.json')); print($c, d['ms_per_step'], d['value'], json.dumps(d['kernel_share']), json.dumps(d['stats'])); ps=d.get('per_size'); print({a:round(b['ms'],2) for a,b in ps.items()} if ps else '')"; done
timeout 900 python bench.py --config 2 --steps 5 --warmup 2 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c2', d['ms_per_step'], d['stats']['steps'])"
for i in 1 2; do timeout 300 python bench.py --steps 10 --no-cpu-baseline --no-secondary 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c1', d['ms_per_step'], d['e2e']['ms_per_step'], json.dumps(d['kernel_share']))"; done
timeout 1500 compute-sanitizer --tool racecheck --racecheck-report hazard --error-exitcode 9 python -m pytest tests/test_gpu_parity.py -q -x -k "heavy_search_spill or exact_mode_warp" > gpurun_out/sanitizer/racecheck.log 2>&1; echo "racecheck rc=$?"; tail -2 gpurun_out/sanitizer/racecheck.log
