#!/bin/bash
# steady-state bench on one B200: GPU parity tests of the new paths, the bench line, the
# full-size --check against the reference; logs under gpurun_out/
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python paper_2604_25899_b200/build.py > gpurun_out/build.log 2>&1
timeout 900 python -m pytest -q -m gpu tests/test_gpu_steady.py tests/test_gpu_l3_order.py 2>&1 | tail -15 > gpurun_out/steady_tests.txt
cat gpurun_out/steady_tests.txt
timeout 900 python bench.py ${BENCH_ARGS} > gpurun_out/bench.out 2> gpurun_out/bench.err
tail -3 gpurun_out/bench.err; cat gpurun_out/bench.out
timeout 1200 python bench.py --check ${CHECK_N:-2} ${CHECK_ARGS} > gpurun_out/check.out 2> gpurun_out/check.err
tail -3 gpurun_out/check.err; tail -4 gpurun_out/check.out
