bash tools/gpu_iter.sh t12 t16
bash tools/gpu_light.sh 16 24 32
