#!/bin/bash
python paper_2604_25899_b200/build.py > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest -q -m gpu -x tests/test_gpu_batch.py tests/test_gpu_steady.py tests/test_gpu_parity.py tests/test_gpu_l3_order.py 2>&1 | tail -1
for cfg in "--k1-grid persistent --k1-gate on" "--k1-grid tasks1 --k1-gate on" "--k1-grid persistent --k1-gate on --k1-after start" "--k1-grid persistent --k1-gate off" "--k1-grid tasks --k1-gate off"; do
  timeout 600 python bench.py --no-cpu-baseline --no-e2e $cfg > gpurun_out/qa.out 2> gpurun_out/qa.err
  python -c "import json;d=json.loads(open('gpurun_out/qa.out').read().strip().splitlines()[-1]);print('$cfg', round(d['value']/1e6,2), round(d['ms_per_step'],3), {k: round(v,3) for k,v in d.get('phase_ms').items()})" || tail -3 gpurun_out/qa.err
done
