#!/bin/bash
set -x
python paper_2604_25899_b200/build.py > gpurun_out/build.log 2>&1
NG=$(nvidia-smi -L | wc -l)
for ka in staged start; do
for n in 1 $NG; do
  timeout 900 python bench.py --gpus $n --no-cpu-baseline --no-e2e --k1-after $ka > gpurun_out/ka_${ka}_n$n.out 2> gpurun_out/ka_${ka}_n$n.err
  python -c "import json;d=json.loads(open('gpurun_out/ka_${ka}_n$n.out').read().strip().splitlines()[-1]);print('$ka', $n, d['value']/1e6, d['ms_per_step'], d.get('phase_ms') or d.get('phase_ms_rank0'))"
done
done
