# round 2 GPU check: the GPU suite, the default bench line (dev tool)
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
timeout 2700 python -m pytest tests -m gpu -q --durations=20 > gpurun_out/t_r2a.log 2>&1; tail -40 gpurun_out/t_r2a.log
timeout 900 python bench.py > gpurun_out/b_r2a.json 2> gpurun_out/b_r2a.err; tail -5 gpurun_out/b_r2a.err; cut -c1-1500 gpurun_out/b_r2a.json
