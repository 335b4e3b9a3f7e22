#!/bin/bash
# ncu --set full of the step kernels (one timed step's worth) after a plain run exited 0
set -x
python paper_2604_25899_b200/build.py > gpurun_out/build.log 2>&1
CMD="python bench.py --profile --steps 3 --warmup 2 --no-cpu-baseline --no-e2e"
$CMD > gpurun_out/plain.log 2>&1 || exit 1
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:'k_(admit|release|route_seq|staged_dir)' --launch-skip 8 --launch-count 6 -o gpurun_out/ncu_step -f $CMD > gpurun_out/ncu_step.log 2>&1
tail -3 gpurun_out/ncu_step.log
