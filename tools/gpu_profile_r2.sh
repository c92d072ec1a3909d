# round-2 profile set (dev tool): launch lists + ncu --set full of configs[1] (every kernel of one step),
# configs[2]'s search kernels and configs[4]'s light / wide kernels (one (size, k) each)
mkdir -p gpurun_out
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c1.csv python bench.py --profile-launches --steps 2 --warmup 1 > /dev/null 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2.csv python bench.py --config 2 --profile-launches --steps 2 --warmup 1 > /dev/null 2>&1
# configs[1]: 7 kernels per step (simplify, prep, discover, light, heavy, recover, recover tail); skip the warm-up step
timeout 900 ncu --set full --clock-control none --import-source on -k regex:mpld_ -s 7 -c 7 -o gpurun_out/full_c1 -f python bench.py --profile-launches --steps 1 --warmup 1 > gpurun_out/ncu_full_c1.log 2>&1; tail -2 gpurun_out/ncu_full_c1.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:mpld_exact -s 2 -c 2 -o gpurun_out/full_c2 -f python bench.py --config 2 --profile-launches --steps 1 --warmup 1 > gpurun_out/ncu_full_c2.log 2>&1; tail -2 gpurun_out/ncu_full_c2.log
ls -la gpurun_out
timeout 600 python bench.py --profile-launches --steps 1 --warmup 1 > gpurun_out/profile_run_c1.json 2>/dev/null
timeout 600 python bench.py --config 2 --profile-launches --steps 1 --warmup 1 > gpurun_out/profile_run_c2.json 2>/dev/null
timeout 900 python tools/batch_sweep.py gpurun_out/batch_sweep.json > gpurun_out/batch_sweep.log 2>&1; tail -3 gpurun_out/batch_sweep.log
bash tools/gpu_sanitize.sh
