# round 2: warp-chunked graph build (dev tool)
mkdir -p gpurun_out/sanitizer
timeout 1200 python -m pytest tests -m gpu -q -x -k "upper or stitch_pairs or capacity or async" > gpurun_out/t_r2p.log 2>&1; tail -3 gpurun_out/t_r2p.log
timeout 900 compute-sanitizer --tool memcheck --error-exitcode 9 python -m pytest tests/test_gpu_parity.py -q -x -k "upper or stitch_pairs" > gpurun_out/sanitizer/memcheck_build.log 2>&1; echo "memcheck rc=$?"; tail -2 gpurun_out/sanitizer/memcheck_build.log
timeout 300 python tools/e2e_probe.py
for i in 1 2; do timeout 300 python bench.py --steps 10 --no-cpu-baseline --no-secondary 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c1', d['ms_per_step'], d['e2e']['ms_per_step'], d['e2e']['h2d_bytes_per_step'])"; done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:graph_build -s 2 -c 1 -o gpurun_out/build -f python tools/build_probe.py > gpurun_out/build.log 2>&1; tail -1 gpurun_out/build.log
