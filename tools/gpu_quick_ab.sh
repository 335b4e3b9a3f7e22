#!/bin/bash
# quick check: eviction/admission GPU tests + steady bench lines (both K1 grids)
python paper_2604_25899_b200/build.py > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest -q -m gpu -x tests/test_gpu_batch.py tests/test_gpu_steady.py tests/test_gpu_parity.py tests/test_gpu_nextuse.py tests/test_gpu_l3_order.py 2>&1 | tail -3
for g in ${GRIDS:-persistent tasks}; do
  timeout 900 python bench.py --no-cpu-baseline --no-e2e --k1-grid $g $EXTRA > gpurun_out/qa.out 2> gpurun_out/qa.err
  python -c "import json;d=json.loads(open('gpurun_out/qa.out').read().strip().splitlines()[-1]);print('$g', round(d['value']/1e6,2), round(d['ms_per_step'],3), {k: round(v,3) for k,v in d.get('phase_ms').items()})"
done
