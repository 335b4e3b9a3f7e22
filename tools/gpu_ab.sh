# A/B of two builds on one box: PYG_SO=libpyg_old.so (experiments) vs the in-tree build
timeout 900 python -m pytest -x -q tests/test_gpu_batch.py tests/test_gpu_parity.py tests/test_gpu_directory.py tests/test_gpu_shard.py tests/test_gpu_prompts.py 2>&1 | tail -2
for v in old new; do
  if [ $v = old ]; then export PYG_SO=/root/repo/libpyg_old.so; else unset PYG_SO; fi
  for w in "deep_research 125000 32" "bursty 125000 32" "bursty 125000 1024" "deep_research 125000 32" "bursty 125000 32"; do
  set -- $w
  timeout 600 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --workload $1 --requests $2 --replicas $3 > gpurun_out/ab_${v}_$1_$3.json 2>gpurun_out/ab_${v}_$1_$3.err
  python -c "import json;d=json.load(open('gpurun_out/ab_${v}_$1_$3.json'));print('$v', '$1', $3, round(d['value']/1e6,2), round(d['ms_per_step'],3), {k:round(v,3) for k,v in d['phase_ms'].items()})"
  done
done
