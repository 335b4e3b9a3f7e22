# usage: NS="1 2" bash tools/gpu_scale.sh   (bench at each N; one JSON line per N into gpurun_out/scale.jsonl)
python paper_2604_25899_b200/build.py > gpurun_out/build.log 2>&1 || exit 1
: > gpurun_out/scale.jsonl
for n in ${NS:-1 2}; do
  if [ "$n" = 1 ]; then
    timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline ${BENCH_ARGS} >> gpurun_out/scale.jsonl 2> gpurun_out/scale_$n.err
  else
    timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $((29600+n)) bench.py --gpus $n --steps 10 --warmup 3 ${BENCH_ARGS} >> gpurun_out/scale.jsonl 2> gpurun_out/scale_$n.err
  fi
  echo "N=$n rc=$?"; grep -v Warning gpurun_out/scale_$n.err | grep -iE "error|Traceback" -A3 | head -20
done
cat gpurun_out/scale.jsonl
