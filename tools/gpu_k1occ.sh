# K1 occupancy A/B: PYG_K1_CTAS_PER_SM=1 (one 8-warp CTA per SM) vs 2
PYG_K1_CTAS_PER_SM=2 timeout 600 python -m pytest tests/test_gpu_batch.py tests/test_gpu_prompts.py -x -q -m gpu 2>&1 | tail -2
for K in 1 2 1 2; do
  for WL in "" "--free-sms -1" "--workload bursty"; do
    PYG_K1_CTAS_PER_SM=$K timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline $WL > gpurun_out/k1o.json 2>/dev/null
    python -c "import json; d=json.load(open('gpurun_out/k1o.json')); print('$K', '$WL', round(d['value']/1e6,2), 'Mreq/s e2e', round(d['e2e']['value']/1e6,2), {k: round(v,3) for k,v in d['phase_ms'].items()})"
  done
done
