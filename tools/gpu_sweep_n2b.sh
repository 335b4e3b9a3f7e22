#!/bin/bash
python paper_2604_25899_b200/build.py > gpurun_out/build.log 2>&1
for cfg in "--k1-grid tasks1 --k1-after staged" "--k1-grid tasks1 --k1-after start" "--k1-grid persistent --k1-after staged"; do
  timeout 600 python bench.py --gpus 2 --no-cpu-baseline --no-e2e $cfg > gpurun_out/qn.out 2> gpurun_out/qn.err
  python -c "import json;d=json.loads(open('gpurun_out/qn.out').read().strip().splitlines()[-1]);print('N=2 [$cfg]', round(d['value']/1e6,2), round(d['ms_per_step'],3), {k: round(v,3) for k,v in d.get('phase_ms_rank0').items()})" || tail -3 gpurun_out/qn.err
done
