#!/bin/bash
# scaling: bench at N = 1, 2, 4 (weak: 125k requests per GPU per step, full lines with e2e)
# + world-2/4 sharded parity tests
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python paper_2604_25899_b200/build.py > gpurun_out/build.log 2>&1
timeout 900 python -m pytest -q -m gpu tests/test_gpu_steady_shard.py tests/test_gpu_shard.py tests/test_gpu_multidevice.py 2>&1 | tail -3
for n in 1 2 4; do
  timeout 900 python bench.py --gpus $n --no-cpu-baseline > gpurun_out/scalef_n$n.json 2> gpurun_out/scalef_n$n.err
  python -c "import json;d=json.loads(open('gpurun_out/scalef_n$n.json').read().strip().splitlines()[-1]);print($n, d['value']/1e6, d['ms_per_step'], d.get('phase_ms'), d.get('e2e',{}).get('value'))"
  timeout 900 python bench.py --gpus $n --impl reference > gpurun_out/scalef_ref_n$n.json 2> gpurun_out/scalef_ref_n$n.err
done
