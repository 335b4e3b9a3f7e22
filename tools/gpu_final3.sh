#!/bin/bash
# final measurement pass (4 GPUs): N=1 full line + reference arm, config 3, N=2/4 with e2e and
# the reference arm, launch list of the N=1 bench
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python paper_2604_25899_b200/build.py > gpurun_out/build.log 2>&1
timeout 900 python bench.py > gpurun_out/f3_n1.json 2> gpurun_out/f3_n1.err
timeout 900 python bench.py --impl reference > gpurun_out/f3_ref_n1.json 2> gpurun_out/f3_ref_n1.err
timeout 900 python bench.py --workload long_context --no-e2e --no-cpu-baseline > gpurun_out/f3_lc.json 2> gpurun_out/f3_lc.err
for n in 2 4; do
  timeout 900 python bench.py --gpus $n --no-cpu-baseline > gpurun_out/f3_n$n.json 2> gpurun_out/f3_n$n.err
  timeout 900 python bench.py --gpus $n --impl reference > gpurun_out/f3_ref_n$n.json 2> gpurun_out/f3_ref_n$n.err
done
CMD="python bench.py --profile --steps 3 --warmup 3 --no-cpu-baseline --no-e2e"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/f3_launches.csv $CMD > gpurun_out/f3_ncu.log 2>&1
for f in gpurun_out/f3_n1.json gpurun_out/f3_n2.json gpurun_out/f3_n4.json gpurun_out/f3_lc.json; do
  python -c "import json;d=json.loads(open('$f').read().strip().splitlines()[-1]);e=d.get('e2e') or {};print('$f', d['n_gpus'], round(d['value']/1e6,2), round(d['ms_per_step'],3), round(d['roofline']['frac'],3), round((e.get('value') or 0)/1e6,2), d.get('clocks'))"
done
