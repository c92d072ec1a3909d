mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:search_heavy -s 2 -c 1 -o gpurun_out/heavy_src -f python tools/greedy_sweep.py 0 1 2 0 > gpurun_out/ncu_hs.log 2>&1; tail -1 gpurun_out/ncu_hs.log
