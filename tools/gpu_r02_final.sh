#!/bin/bash
# round-2 final measurement pass on one B200: bench line (baselines + e2e), reference arm,
# config-3 line, launch list of the bench, ncu --set full of the top kernels
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks_throttle_reasons.active --format=csv
python paper_2604_25899_b200/build.py > gpurun_out/build.log 2>&1
timeout 900 python bench.py > gpurun_out/final_bench.json 2> gpurun_out/final_bench.err; tail -2 gpurun_out/final_bench.err
timeout 900 python bench.py --impl reference > gpurun_out/final_ref.json 2> gpurun_out/final_ref.err; tail -2 gpurun_out/final_ref.err
timeout 900 python bench.py --workload long_context --no-e2e --no-cpu-baseline > gpurun_out/final_lc.json 2> gpurun_out/final_lc.err
CMD="python bench.py --profile --steps 3 --warmup 2 --no-cpu-baseline --no-e2e"
$CMD > gpurun_out/plain.log 2>&1 || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/final_launches.csv $CMD > gpurun_out/ncu_launches.log 2>&1
for k in k_hash_staged k_admit k_route_seq; do
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:"$k" --launch-skip 3 --launch-count 1 \
    -o gpurun_out/final_ncu_$k -f $CMD > gpurun_out/ncu_$k.log 2>&1
  tail -1 gpurun_out/ncu_$k.log
done
