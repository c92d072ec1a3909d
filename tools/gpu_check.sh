set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -15
timeout 120 python __graft_entry__.py smoke 2>&1 | tail -3
timeout 300 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -3 gpurun_out/bench.err; cat gpurun_out/bench.json
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --profile-launches --steps 2 --warmup 1 > /dev/null 2>&1
timeout 300 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/ref.json 2>/dev/null; cat gpurun_out/ref.json
