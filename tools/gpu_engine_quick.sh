#!/bin/bash
# engine whole-trace parity at WF workflows with the adapter call profile, + GPU tests
set -x
python paper_2604_25899_b200/build.py > gpurun_out/build.log 2>&1
timeout 900 python -m pytest -q -m gpu ${TESTS:-tests/test_gpu_engine.py tests/test_gpu_parity.py tests/test_gpu_dropin.py} 2>&1 | tail -5
WF=${WF:-200}; s=${SEED:-1}
mkdir -p gpurun_out/q/ref gpurun_out/q/b200
( t0=$(date +%s%N); ./oracle/_ref/engine_ref16 gpurun_out/q/ref $WF $s > gpurun_out/q/ref.out 2>&1; echo "ref rc=$? wall_ms $(( ($(date +%s%N) - t0) / 1000000 ))" >> gpurun_out/q/ref.out ) &
t0=$(date +%s%N); PYG_ADAPTER_PROFILE=1 PYG_ENGINE_MAX_REPLICAS=1024 ./integration/_build/engine_b200 gpurun_out/q/b200 $WF $s > gpurun_out/q/b200.out 2>&1; echo "b200 rc=$? wall_ms $(( ($(date +%s%N) - t0) / 1000000 ))" >> gpurun_out/q/b200.out
wait
cat gpurun_out/q/ref.out; head -25 gpurun_out/q/b200.out; tail -2 gpurun_out/q/b200.out
for f in event_log.txt routing_log.jsonl cache_log.jsonl scale_log.jsonl metrics.json; do
  if cmp -s gpurun_out/q/ref/$f gpurun_out/q/b200/$f; then echo "IDENTICAL $f $(wc -l < gpurun_out/q/ref/$f)"; else echo "DIFFER $f"; fi
done
rm -rf gpurun_out/q/ref gpurun_out/q/b200
