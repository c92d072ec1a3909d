mkdir -p gpurun_out
MPLD_LIB=paper_2303_14335_b200/lib/variants/libmpld_diag.so timeout 300 python tools/heavy_trace.py 2 > gpurun_out/heavy_trace.log 2>&1; head -12 gpurun_out/heavy_trace.log
for i in 1 2; do timeout 120 python tools/greedy_sweep.py 0 1 2 0 2>&1 | tail -1 | cut -c1-200; done
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "exact or heavy or config2 or stress" > gpurun_out/t_heavy.log 2>&1; tail -2 gpurun_out/t_heavy.log
