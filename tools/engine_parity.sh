# whole-trace parity: the reference engine with its CPU cache/router vs the same engine on the
# B200 backend (integration/_build/engine_b200); usage: WF=20 SEED=1 bash tools/engine_parity.sh
WF=${WF:-20}; SEED=${SEED:-1}
mkdir -p gpurun_out/eng_ref gpurun_out/eng_b200
./oracle/_ref/engine_ref16 gpurun_out/eng_ref $WF $SEED
t0=$(date +%s); ./integration/_build/engine_b200 gpurun_out/eng_b200 $WF $SEED; echo "b200 engine rc=$? wall $(( $(date +%s) - t0 )) s"
for f in event_log.txt routing_log.jsonl cache_log.jsonl scale_log.jsonl metrics.json; do
  if cmp -s gpurun_out/eng_ref/$f gpurun_out/eng_b200/$f; then echo "IDENTICAL $f $(wc -l < gpurun_out/eng_ref/$f) lines"; else echo "DIFFER $f"; diff gpurun_out/eng_ref/$f gpurun_out/eng_b200/$f | head -5; fi
done
rm -f gpurun_out/eng_*/cache_log.jsonl
