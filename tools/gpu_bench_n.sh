#!/bin/bash
# bench at N = 1 and N = #GPUs (no baselines), then the N=1 launch list (ncu, serialized)
set -x
NG=$(nvidia-smi -L | wc -l)
python paper_2604_25899_b200/build.py > gpurun_out/build.log 2>&1
for n in 1 $NG; do
  timeout 900 python bench.py --gpus $n --no-cpu-baseline --no-e2e ${BENCH_ARGS} > gpurun_out/bench_n$n.out 2> gpurun_out/bench_n$n.err
  echo "rc=$?"; tail -3 gpurun_out/bench_n$n.err
  python -c "import json;d=json.load(open('gpurun_out/bench_n$n.out'));print($n, d['value']/1e6, d['ms_per_step'], d.get('phase_ms'), d['config']['placed_per_step'])"
done
if [ "${LAUNCHES:-1}" = "1" ]; then
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:'k_(hash_staged|len_keys|staged|node|gs_init|seq|chunk|super|group|route|rep_|placed|iota|admit|l3_|release|nodes_compose|reg_set_batch|clamp)|Radix|Scan' --launch-skip 60 -c 300 --csv --log-file gpurun_out/launches.csv python bench.py --profile --steps 3 --warmup 2 > gpurun_out/ncu_launch.log 2>&1
python tools/launches_summary.py gpurun_out/launches.csv | head -40
fi
