# K2 warp walks: parity + A/B of staged-matrix time (PYG_K2_WARP_MIN huge = one thread per walk)
python paper_2604_25899_b200/build.py > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_directory.py tests/test_gpu_batch.py tests/test_gpu_stage.py -x -q -m gpu 2>&1 | tail -3
run() {
  PYG_K2_WARP_MIN=$1 timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e $2 > gpurun_out/k2.json 2>/dev/null
  python -c "import json,sys; d=json.load(open('gpurun_out/k2.json')); print('$1', '$2', round(d['value']/1e6,2), 'Mreq/s', {k: round(v,3) for k,v in d['phase_ms'].items()})"
}
for W in 2000000000 64 128 256 512; do
  for WL in "" "--workload bursty"; do run $W "$WL"; done
done
for W in 2000000000 128; do run $W "--workload bursty --replicas 1024"; run $W "--workload bursty --requests 16000"; done
