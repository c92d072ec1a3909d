for v in default prespill; do L=""; [ $v != default ] && L=paper_2303_14335_b200/lib/variants/libmpld_$v.so; MPLD_LIB=$L timeout 600 ncu --set full --clock-control none --import-source on -k regex:"mpld_exact_cover_search_heavy" -c 1 -o gpurun_out/heavy_$v -f python bench.py --profile-launches --steps 1 --warmup 1 > /dev/null 2>&1; done
ls gpurun_out
