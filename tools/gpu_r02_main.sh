#!/bin/bash
# round-2 measurement pass on one B200: full bench line (baselines + e2e), --check at full
# size, config-3 bench, free-SM sweep, then config-1 engine parity at 1,000 workflows x 3 seeds
set -x
python paper_2604_25899_b200/build.py > gpurun_out/build.log 2>&1
timeout 900 python bench.py > gpurun_out/bench_full.out 2> gpurun_out/bench_full.err; tail -2 gpurun_out/bench_full.err
timeout 1200 python bench.py --check 3 > gpurun_out/check3.out 2> gpurun_out/check3.err; tail -2 gpurun_out/check3.err; tail -1 gpurun_out/check3.out | cut -c1-300
timeout 900 python bench.py --workload long_context --no-e2e --no-cpu-baseline > gpurun_out/bench_lc.out 2> gpurun_out/bench_lc.err; tail -2 gpurun_out/bench_lc.err
timeout 1200 python bench.py --workload long_context --check 2 > gpurun_out/check_lc.out 2> gpurun_out/check_lc.err; tail -1 gpurun_out/check_lc.out | cut -c1-300
for fs in 0 24 48; do
  timeout 600 python bench.py --no-e2e --no-cpu-baseline --free-sms $fs > gpurun_out/bench_fs$fs.out 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/bench_fs$fs.out'));print('free_sms', $fs, d['value']/1e6, d['ms_per_step'], d['phase_ms'])"
done
bash tools/gpu_engine1000.sh
