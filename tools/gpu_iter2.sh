#!/bin/bash
# full GPU suite + bench config 4 / config 3 + K1 sweep
set -x
python paper_2604_25899_b200/build.py > gpurun_out/build.log 2>&1
timeout 1500 python -m pytest -q -m gpu tests 2>&1 | tail -8 > gpurun_out/gpu_tests.txt; cat gpurun_out/gpu_tests.txt
for w in bursty long_context; do
  timeout 900 python bench.py --workload $w --no-e2e --no-cpu-baseline > gpurun_out/bench_$w.out 2> gpurun_out/bench_$w.err
  python -c "import json;d=json.load(open('gpurun_out/bench_$w.out'));print('$w', d['value']/1e6, d['ms_per_step'], d['phase_ms'], d['config']['placed_per_step'], d['roofline']['frac'])"
done
timeout 600 python tools/k1_sweep.py --splits -1,0 > gpurun_out/k1_sweep.jsonl 2>&1; cat gpurun_out/k1_sweep.jsonl
