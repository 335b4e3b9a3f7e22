set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python paper_2604_25899_b200/build.py > gpurun_out/build.log 2>&1
timeout 1200 python -m pytest tests -x -q -m gpu ${PYTEST_ARGS} 2>&1 | tail -40
