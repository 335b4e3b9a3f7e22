# config-5 style sweep on one GPU: bursty prompt distribution, R requests x N replicas
python paper_2604_25899_b200/build.py > gpurun_out/build.log 2>&1
: > gpurun_out/sweep.jsonl
for pt in "1000 8" "16000 32" "125000 32" "125000 256" "125000 1024" "500000 256"; do
  set -- $pt
  timeout 600 python bench.py --workload bursty --requests $1 --replicas $2 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline >> gpurun_out/sweep.jsonl 2> gpurun_out/sweep_$1_$2.err
  echo "R=$1 N=$2 rc=$?"
done
