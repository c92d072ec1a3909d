# recovery tuning sweep (dev tool): level trace + step time per variant library
mkdir -p gpurun_out/lev
for rep in 1 2; do
for v in default p2 minb2 cti2 cti4 nb8 nb2; do
  if [ $v = default ]; then unset MPLD_LIB; else export MPLD_LIB=$PWD/paper_2303_14335_b200/lib/variants/libmpld_$v.so; fi
  for c in 1 3; do timeout 300 python tools/level_trace.py $c >> gpurun_out/lev/trace.jsonl 2>> gpurun_out/lev/err.log; done
done; done
echo done
