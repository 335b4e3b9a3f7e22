#!/bin/bash
# K1 warps-per-CTA experiment: K1 alone on config-4 bursts, then the steady bench.
python paper_2604_25899_b200/build.py > gpurun_out/build.log 2>&1
for w in 8 12 16; do
  PYG_K1_WARPS=$w timeout 600 python tools/k1_sweep.py --sizes 16000,125000 --splits -1 | sed "s/^/W=$w /"
done
for w in 8 16; do
  for g in persistent tasks; do
    PYG_K1_WARPS=$w timeout 900 python bench.py --no-cpu-baseline --no-e2e --k1-grid $g > gpurun_out/kw.out 2> gpurun_out/kw.err
    python -c "import json;d=json.loads(open('gpurun_out/kw.out').read().strip().splitlines()[-1]);print('W=$w $g', round(d['value']/1e6,2), round(d['ms_per_step'],3), {k: round(v,3) for k,v in d.get('phase_ms').items()})"
  done
done
