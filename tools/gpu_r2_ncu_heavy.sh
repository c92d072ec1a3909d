mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none -k regex:search_heavy -s 2 -c 1 -o gpurun_out/heavy_whole -f python tools/greedy_sweep.py 0 1 2 0 > gpurun_out/ncu_hw.log 2>&1; tail -1 gpurun_out/ncu_hw.log
timeout 600 ncu --set full --clock-control none -k regex:search_heavy -s 4 -c 1 -o gpurun_out/heavy_tile -f python tools/greedy_sweep.py 0 1 2 2 > gpurun_out/ncu_ht.log 2>&1; tail -1 gpurun_out/ncu_ht.log
