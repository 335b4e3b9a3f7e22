#!/bin/bash
# full GPU suite + one bench line (no baselines)
set -x
python paper_2604_25899_b200/build.py > gpurun_out/build.log 2>&1
timeout 1500 python -m pytest -q -m gpu tests ${PYTEST_ARGS} 2>&1 | tail -25 > gpurun_out/gpu_tests.txt
cat gpurun_out/gpu_tests.txt
timeout 600 python bench.py --no-cpu-baseline --no-e2e ${BENCH_ARGS} > gpurun_out/bench.out 2> gpurun_out/bench.err
tail -3 gpurun_out/bench.err
python -c "import json;d=json.load(open('gpurun_out/bench.out'));print(d['value']/1e6, d['ms_per_step'], d['phase_ms'], d['config']['placed_per_step'], d['config']['evicted_blocks_per_step'], d['roofline']['frac'])"
