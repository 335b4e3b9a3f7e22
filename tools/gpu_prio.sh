#!/bin/bash
python -c "import torch; print('priority range', torch.cuda.Stream.priority_range())"
for p in -1 -2 -3 -5; do
  PYG_STEP_PRIORITY=$p timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/qa.out 2> gpurun_out/qa.err
  python -c "import json;d=json.loads(open('gpurun_out/qa.out').read().strip().splitlines()[-1]);print('prio $p', round(d['value']/1e6,2), round(d['ms_per_step'],3), {k: round(v,3) for k,v in d.get('phase_ms').items()})" || tail -3 gpurun_out/qa.err
done
