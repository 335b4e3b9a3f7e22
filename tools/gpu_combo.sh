bash tools/gpu_ab.sh
bash tools/gpu_e2e2.sh
