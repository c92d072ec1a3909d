# round 2 re-entry check (dev tool): full GPU suite, smoke, default bench line, config 2 line
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
timeout 2400 python -m pytest tests -m gpu -q -x --durations=15 > gpurun_out/t_full.log 2>&1; echo "pytest rc=$?"; tail -25 gpurun_out/t_full.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo "bench rc=$?"; tail -c 3000 gpurun_out/bench_default.json; tail -5 gpurun_out/bench_default.err
