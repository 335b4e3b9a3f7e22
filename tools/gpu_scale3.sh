#!/bin/bash
set -x
python paper_2604_25899_b200/build.py > gpurun_out/build.log 2>&1
timeout 900 python -m pytest -q -m gpu tests/test_gpu_steady_shard.py tests/test_gpu_shard.py 2>&1 | tail -3
bash tools/gpu_scale2.sh 2>&1 | grep -v "^+"
