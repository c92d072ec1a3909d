# round 2: light budget sweep (exact mode hand-off point) on configs[1] and [2] (dev tool)
for ls in 16 32 48 96; do
  for c in 1 2; do
    MPLD_LIGHT_STEPS=$ls timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-secondary 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('light', $ls, 'c$c', round(d['ms_per_step'],4), d['stats']['steps'], {k: round(v,3) for k,v in d['kernel_share'].items()})"
  done
done
