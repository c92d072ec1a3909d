# compute-sanitizer over the search tests (dev tool): memcheck, racecheck, synccheck
mkdir -p gpurun_out/sanitizer
T="tests/test_gpu_parity.py"
SEL="edge_cases or heavy_search_spill or exact_mode_warp or stitch_pairs or sharded or recovery_cluster_tail or k4_budget"
timeout 1500 compute-sanitizer --tool memcheck --error-exitcode 9 python -m pytest $T -q -x -k "$SEL" > gpurun_out/sanitizer/memcheck.log 2>&1; echo "memcheck rc=$?"; tail -3 gpurun_out/sanitizer/memcheck.log
timeout 1500 compute-sanitizer --tool racecheck --racecheck-report hazard --error-exitcode 9 python -m pytest $T -q -x -k "heavy_search_spill or exact_mode_warp" > gpurun_out/sanitizer/racecheck.log 2>&1; echo "racecheck rc=$?"; tail -3 gpurun_out/sanitizer/racecheck.log
timeout 900 compute-sanitizer --tool synccheck --error-exitcode 9 python -m pytest $T -q -x -k "heavy_search_spill or exact_mode_warp" > gpurun_out/sanitizer/synccheck.log 2>&1; echo "synccheck rc=$?"; tail -3 gpurun_out/sanitizer/synccheck.log
