#!/bin/bash
set -x
python paper_2604_25899_b200/build.py > gpurun_out/build.log 2>&1
NG=$(nvidia-smi -L | wc -l)
for n in 2 4; do
  [ $n -le $NG ] || continue
  timeout 900 python bench.py --gpus $n --no-cpu-baseline --no-e2e ${BENCH_ARGS} > gpurun_out/scale_n$n.out 2> gpurun_out/scale_n$n.err
  python -c "import json;d=json.loads(open('gpurun_out/scale_n$n.out').read().strip().splitlines()[-1]);print($n, d['value']/1e6, d['ms_per_step'], d.get('phase_ms_rank0'), d.get('hash_ms_rank0'))"
done
