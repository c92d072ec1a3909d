# round 2: build prefix sums in parallel, packed recovery state, pair bound off (dev tool)
mkdir -p gpurun_out/sanitizer
timeout 2400 python -m pytest tests -m gpu -q -x > gpurun_out/t_r2o.log 2>&1; tail -3 gpurun_out/t_r2o.log
timeout 300 python tools/e2e_probe.py
for i in 1 2; do timeout 900 python bench.py --config 2 --steps 5 --warmup 2 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c2', d['ms_per_step'], d['stats']['steps'], d['kernel_share']['mpld_exact_cover_search_heavy'])"; done
for i in 1 2 3; do timeout 300 python bench.py --steps 10 --no-cpu-baseline --no-secondary 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c1', d['ms_per_step'], d['e2e']['ms_per_step'], d['e2e']['h2d_bytes_per_step'], json.dumps({k: round(v,3) for k,v in d['kernel_share'].items()}))"; done
timeout 300 python tools/kernel_times.py 2>&1 | tail -3
