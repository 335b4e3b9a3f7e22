#!/bin/bash
set -x
python paper_2604_25899_b200/build.py > gpurun_out/build.log 2>&1
timeout 600 python -m pytest -q -m gpu tests/test_gpu_batch.py -k hash 2>&1 | tail -2
for cfg in "--k1-grid tasks --k1-after start" "--k1-grid tasks --k1-after staged" "--k1-grid persistent --k1-after start"; do
  timeout 900 python bench.py --no-cpu-baseline --no-e2e $cfg > gpurun_out/kg.out 2> gpurun_out/kg.err
  python -c "import json;d=json.loads(open('gpurun_out/kg.out').read().strip().splitlines()[-1]);print('$cfg', d['value']/1e6, d['ms_per_step'], d.get('phase_ms'))"
done
