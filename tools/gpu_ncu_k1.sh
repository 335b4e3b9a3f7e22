#!/bin/bash
# ncu --set full of K1 alone on one config-4 burst (125k requests), adaptive split on / off
python paper_2604_25899_b200/build.py > gpurun_out/build.log 2>&1
for sp in -1 0; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_hash_staged -s 2 -c 1 \
    -o gpurun_out/k1_bursty_split$sp python tools/k1_sweep.py --sizes 125000 --splits $sp --grids persistent > gpurun_out/ncu_k1_$sp.log 2>&1
  tail -3 gpurun_out/ncu_k1_$sp.log
done
