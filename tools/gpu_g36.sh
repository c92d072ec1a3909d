timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for p in 1 0 1 0; do MPLD_PDL=$p timeout 300 python bench.py --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('pdl', $p, round(d['ms_per_step'],4), d['gpu_launches'], {k: round(v,3) for k,v in d['kernel_share'].items()})"; done
