# round 2: full default bench line (headline + secondary), sanitizers (dev tool)
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/b_r2h.json 2> gpurun_out/b_r2h.err; tail -3 gpurun_out/b_r2h.err; cut -c1-600 gpurun_out/b_r2h.json
bash tools/gpu_sanitize.sh
