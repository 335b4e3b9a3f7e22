# A/B of two builds on one box: PYG_SO=libpyg_old.so (experiments) vs the in-tree build
timeout 900 python -m pytest -x -q tests/test_gpu_batch.py tests/test_gpu_prompts.py 2>&1 | tail -2
for v in old new; do
  if [ $v = old ]; then export PYG_SO=/root/repo/libpyg_old.so; else unset PYG_SO; fi
  for w in deep_research bursty; do
  timeout 600 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --workload $w ${AB_ARGS} > gpurun_out/ab_${v}_$w.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/ab_${v}_$w.json'));print('$v', '$w', round(d['value']/1e6,1), round(d['ms_per_step'],3), {k:round(v,3) for k,v in d['phase_ms'].items()})"
  done
done
