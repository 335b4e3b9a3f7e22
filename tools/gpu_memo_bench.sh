#!/bin/bash
python paper_2604_25899_b200/build.py > gpurun_out/build.log 2>&1
for cfg in "--k1-grid persistent --k1-after start --free-sms 24 --k1-memo on" "--k1-grid persistent --k1-after start --free-sms 8 --k1-memo on" "--k1-grid persistent --k1-after start --free-sms 24" ""; do
  timeout 600 python bench.py --no-cpu-baseline --no-e2e $cfg > gpurun_out/qa.out 2> gpurun_out/qa.err
  python -c "import json;d=json.loads(open('gpurun_out/qa.out').read().strip().splitlines()[-1]);print('cfg [$cfg]', round(d['value']/1e6,2), round(d['ms_per_step'],3), {k: round(v,3) for k,v in d.get('phase_ms').items()})" || tail -3 gpurun_out/qa.err
done
