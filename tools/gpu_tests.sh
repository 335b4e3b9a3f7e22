#!/bin/bash
# full -m gpu suite on whatever GPUs the box has; log under gpurun_out/
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python paper_2604_25899_b200/build.py > gpurun_out/build.log 2>&1
timeout ${TEST_TIMEOUT:-1500} python -m pytest tests -q -m gpu ${PYTEST_ARGS} 2>&1 | tail -60 > gpurun_out/gpu_tests.txt
cat gpurun_out/gpu_tests.txt | tail -30
