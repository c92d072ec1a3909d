# phase breakdown + one ncu --set full capture of the graph kernels (dev tool)
timeout 300 python tools/kernel_times.py --replicas 16 --single 2>&1 | tail -8
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"mpld_(simplify|recover)" -c 2 -o gpurun_out/graph_full -f python bench.py --profile-launches --steps 1 --warmup 1 > gpurun_out/ncu_graph.log 2>&1; tail -3 gpurun_out/ncu_graph.log
