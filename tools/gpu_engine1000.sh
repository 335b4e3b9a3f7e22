#!/bin/bash
# config 1 whole-trace parity at 1,000 workflows, seeds 1-3: the reference engine on its own
# cache/router vs the same engine on the B200 backend; wall times of both
set -x
python paper_2604_25899_b200/build.py > gpurun_out/build.log 2>&1
make -s -C oracle restated > /dev/null 2>&1
WF=${WF:-1000}
for s in ${SEEDS:-1 2 3}; do
  mkdir -p gpurun_out/e$s/ref gpurun_out/e$s/b200
  ( t0=$(date +%s%N); ./oracle/_ref/engine_ref16 gpurun_out/e$s/ref $WF $s > gpurun_out/e$s/ref.out 2>&1; echo "ref rc=$? wall_ms $(( ($(date +%s%N) - t0) / 1000000 ))" >> gpurun_out/e$s/ref.out ) &
done
for s in ${SEEDS:-1 2 3}; do
  t0=$(date +%s%N); PYG_ENGINE_MAX_REPLICAS=${MAXREP:-1024} ./integration/_build/engine_b200 gpurun_out/e$s/b200 $WF $s > gpurun_out/e$s/b200.out 2>&1; echo "b200 rc=$? wall_ms $(( ($(date +%s%N) - t0) / 1000000 ))" >> gpurun_out/e$s/b200.out
done
wait
for s in ${SEEDS:-1 2 3}; do
  echo "== seed $s"; cat gpurun_out/e$s/ref.out gpurun_out/e$s/b200.out
  for f in event_log.txt routing_log.jsonl cache_log.jsonl scale_log.jsonl metrics.json; do
    if cmp -s gpurun_out/e$s/ref/$f gpurun_out/e$s/b200/$f; then echo "IDENTICAL $f $(wc -l < gpurun_out/e$s/ref/$f) lines $(md5sum < gpurun_out/e$s/ref/$f | cut -c1-16)"; else echo "DIFFER $f"; fi
  done
  rm -rf gpurun_out/e$s/ref gpurun_out/e$s/b200
done
