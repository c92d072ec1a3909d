# round profile set: bench lines (configs 1-3), ncu launch list, ncu --set full of every kernel of one step (dev tool)
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 300 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -2 gpurun_out/bench.err; cat gpurun_out/bench.json
for c in 2 3; do timeout 600 python bench.py --config $c --steps 5 > gpurun_out/bench_c$c.json 2> gpurun_out/bench_c$c.err; tail -1 gpurun_out/bench_c$c.err; cut -c1-300 gpurun_out/bench_c$c.json; done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --profile-launches --steps 2 --warmup 1 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:mpld_ -c 9 -o gpurun_out/full -f python bench.py --profile-launches --steps 1 --warmup 1 > gpurun_out/ncu_full.log 2>&1; tail -2 gpurun_out/ncu_full.log
