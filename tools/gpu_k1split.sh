#!/bin/bash
# K1 split tasks: parity, the bench at several split thresholds, ncu of the admission kernel
set -x
python paper_2604_25899_b200/build.py > gpurun_out/build.log 2>&1
timeout 900 python -m pytest -q -m gpu tests/test_gpu_batch.py -k hash tests/test_gpu_steady.py 2>&1 | tail -15 > gpurun_out/k1_tests.txt
cat gpurun_out/k1_tests.txt
for sm in 8192 4096 16384 0; do
  timeout 600 python bench.py --no-cpu-baseline --no-e2e --split-min $sm > gpurun_out/bench_split_$sm.out 2> gpurun_out/bench_split_$sm.err
  python -c "import json;d=json.load(open('gpurun_out/bench_split_$sm.out'));print($sm, d['value']/1e6, d['ms_per_step'], d['phase_ms'], d['config']['placed_per_step'], d['config']['evicted_blocks_per_step'])"
done
timeout 900 ncu --kernel-name regex:k_admit --launch-skip 4 --launch-count 1 --set full --import-source on --clock-control none -o gpurun_out/ncu_admit -f python bench.py --profile --steps 3 --warmup 2 > gpurun_out/ncu_admit.log 2>&1
tail -3 gpurun_out/ncu_admit.log
