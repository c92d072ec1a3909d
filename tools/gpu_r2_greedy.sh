mkdir -p gpurun_out
for fl in 0 2; do timeout 120 python tools/greedy_sweep.py 0 1 2 $fl 2>&1 | tail -1; done > gpurun_out/greedy6.log
for fl in 0; do timeout 120 python tools/greedy_sweep.py 0 1 1 $fl 2>&1 | tail -1; done >> gpurun_out/greedy6.log
cat gpurun_out/greedy6.log | python -c "
import sys, json
for l in sys.stdin:
    try: d = json.loads(l)
    except Exception: print(l.strip()[:200]); continue
    print(d['flags'], d['heavy_us'], d['steps'], d['heavy_comps'], d['heavy_nodes'], d['kernels'])"
