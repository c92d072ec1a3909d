# simplification tail tuning sweep (dev tool): step time per variant library
mkdir -p gpurun_out/lev2
for rep in 1 2; do
for v in default cr1 tail256 tail4k grp8 grp32; do
  if [ $v = default ]; then unset MPLD_LIB; else export MPLD_LIB=$PWD/paper_2303_14335_b200/lib/variants/libmpld_$v.so; fi
  for c in 1 3; do timeout 300 python tools/level_trace.py $c >> gpurun_out/lev2/trace.jsonl 2>> gpurun_out/lev2/err.log; done
done; done
echo done
