# ncu --set full capture of the heavy search kernel with source (dev tool)
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"mpld_exact_cover_search_heavy" -c 1 -o gpurun_out/heavy_full -f python bench.py --profile-launches --steps 1 --warmup 1 > gpurun_out/ncu_heavy.log 2>&1; tail -3 gpurun_out/ncu_heavy.log
