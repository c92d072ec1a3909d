bash tools/gpu_iter.sh t4 t8 t4d2
bash tools/gpu_ncu_heavy.sh
