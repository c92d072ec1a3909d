# end-of-round checks (dev tool): smoke, shard-mode bench on one GPU, the reference arm, a short default bench
timeout 120 python __graft_entry__.py smoke 2>&1 | tail -1
MPLD_BENCH_MODE=shard timeout 300 python bench.py --mode shard --config 3 --steps 3 --no-cpu-baseline 2>&1 | tail -1 | cut -c1-300
timeout 300 python bench.py --impl reference --steps 3 --warmup 3 2>/dev/null | cut -c1-300
timeout 300 python bench.py --steps 5 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],4), d['e2e']['value'], d['gpu_launches'], d['roofline']['kernel'], round(d['roofline']['frac'],4))"
