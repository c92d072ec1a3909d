# round 2: CAS ring claims restored (dev tool)
mkdir -p gpurun_out/sanitizer
timeout 2400 python -m pytest tests -m gpu -q -x -k "exact or spill or config2 or k4 or stress or sharded or capacity" > gpurun_out/t_r2j.log 2>&1; tail -3 gpurun_out/t_r2j.log
for i in 1 2 3; do timeout 900 python bench.py --config 2 --steps 5 --warmup 2 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c2', d['ms_per_step'], d['stats']['steps'], d['kernel_share']['mpld_exact_cover_search_heavy'])"; done
timeout 1500 compute-sanitizer --tool racecheck --racecheck-report hazard --error-exitcode 9 python -m pytest tests/test_gpu_parity.py -q -x -k "heavy_search_spill or exact_mode_warp" > gpurun_out/sanitizer/racecheck.log 2>&1; echo "racecheck rc=$?"; tail -2 gpurun_out/sanitizer/racecheck.log
