mkdir -p gpurun_out
for i in 1 2 3; do timeout 120 python tools/greedy_sweep.py 0 1 2 0 2>&1 | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(d['heavy_us'], d['steps'])"; done
MPLD_LIB=paper_2303_14335_b200/lib/variants/libmpld_diag.so timeout 300 python tools/heavy_trace.py 2 2>&1 | head -4
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "exact or heavy or config2 or spill" > gpurun_out/t_heavy.log 2>&1; tail -2 gpurun_out/t_heavy.log
