#!/bin/bash
# scaling: bench at N = 1, 2, 4 (weak: 125k requests per GPU per step) + world-4 parity
set -x
python paper_2604_25899_b200/build.py > gpurun_out/build.log 2>&1
NG=$(nvidia-smi -L | wc -l)
timeout 900 python -m pytest -q -m gpu tests/test_gpu_steady_shard.py tests/test_gpu_shard.py 2>&1 | tail -3
for n in 1 2 4; do
  [ $n -le $NG ] || continue
  timeout 900 python bench.py --gpus $n --no-cpu-baseline --no-e2e ${BENCH_ARGS} > gpurun_out/scale_n$n.out 2> gpurun_out/scale_n$n.err
  python -c "import json;d=json.load(open('gpurun_out/scale_n$n.out'));print($n, d['value']/1e6, d['ms_per_step'], d.get('phase_ms'), d['config']['placed_per_step'])"
done
python tools/k1_sweep.py --sizes=1000,16000,125000 --splits=-1 2>&1 | tail -3
python tools/k1_sweep.py --workload long_context --sizes=12500 --splits=-1 2>&1 | tail -1
