bash tools/gpu_iter.sh diag
timeout 300 python bench.py --no-cpu-baseline 2>/dev/null | cut -c1-400
