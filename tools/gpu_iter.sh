#!/bin/bash
# one iteration: targeted GPU tests, bench N=1 (no baselines), ncu --set full of the step kernels
set -x
python paper_2604_25899_b200/build.py > gpurun_out/build.log 2>&1
timeout 900 python -m pytest -q -m gpu ${TESTS:-tests/test_gpu_parity.py tests/test_gpu_batch.py tests/test_gpu_steady.py tests/test_gpu_l3_order.py tests/test_golden.py} 2>&1 | tail -15 > gpurun_out/iter_tests.txt
tail -4 gpurun_out/iter_tests.txt
timeout 600 python bench.py --no-cpu-baseline --no-e2e ${BENCH_ARGS} > gpurun_out/bench.out 2> gpurun_out/bench.err || tail -5 gpurun_out/bench.err
python -c "import json;d=json.load(open('gpurun_out/bench.out'));print(d['value']/1e6, d['ms_per_step'], d['phase_ms'], d['config']['placed_per_step'], d['config']['evicted_blocks_per_step'])"
if [ "${NCU:-1}" = "1" ]; then
CMD="python bench.py --profile --steps 3 --warmup 2 --no-cpu-baseline --no-e2e ${BENCH_ARGS}"
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:"${NCU_K:-k_(admit|release|route_seq|staged_dir)}" --launch-skip ${NCU_SKIP:-8} --launch-count ${NCU_N:-6} -o gpurun_out/ncu_step -f $CMD > gpurun_out/ncu_step.log 2>&1
tail -2 gpurun_out/ncu_step.log
fi
