# ncu --set full of the tile pipeline's kernels on configs[1] (dev tool)
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"piece_order|tile_decompose" -s 3 -c 3 -o gpurun_out/tile_c1 -f python bench.py --profile-launches --steps 1 --warmup 1 > gpurun_out/ncu_tile_c1.log 2>&1; tail -3 gpurun_out/ncu_tile_c1.log
