#!/bin/bash
# ncu --set full of each step kernel (one launch after warm-up) after a plain run exited 0
set -x
python paper_2604_25899_b200/build.py > gpurun_out/build.log 2>&1
CMD="python bench.py --profile --steps 3 --warmup 2 --no-cpu-baseline --no-e2e $EXTRA"
$CMD > gpurun_out/plain.log 2>&1 || exit 1
for k in ${KERNELS:-k_route_seq k_admit k_staged_dir k_release k_hash_staged}; do
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:"$k" --launch-skip 3 --launch-count 1 \
    -o gpurun_out/r02_ncu_$k -f $CMD > gpurun_out/ncu_$k.log 2>&1
  tail -2 gpurun_out/ncu_$k.log
done
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_step.csv $CMD > gpurun_out/ncu_launches.log 2>&1
tail -2 gpurun_out/ncu_launches.log
