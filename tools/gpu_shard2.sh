#!/bin/bash
# sharded steady step: parity (world 1/2[/4]) + bench at N = 1 and N = #GPUs
set -x
NG=$(nvidia-smi -L | wc -l)
python paper_2604_25899_b200/build.py > gpurun_out/build.log 2>&1
timeout 1200 python -m pytest -q -m gpu tests/test_gpu_steady_shard.py tests/test_gpu_shard.py 2>&1 | tail -30 > gpurun_out/shard_tests.txt
cat gpurun_out/shard_tests.txt | tail -5
for n in 1 $NG; do
  timeout 900 python bench.py --gpus $n --no-cpu-baseline --no-e2e > gpurun_out/bench_n$n.out 2> gpurun_out/bench_n$n.err
  tail -2 gpurun_out/bench_n$n.err
  python -c "import json;d=json.load(open('gpurun_out/bench_n$n.out'));print($n, d['value']/1e6, d['ms_per_step'], d.get('phase_ms'), d['config']['placed_per_step'])"
done
