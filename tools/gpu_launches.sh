set -x
python paper_2604_25899_b200/build.py > gpurun_out/build.log 2>&1
CMD="python bench.py --steps 3 --warmup 1 --profile --no-e2e --no-cpu-baseline"
$CMD > gpurun_out/plain2.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:'k_(hash_staged|len|staged|node|gs|seq|group|route|rep|placed|iota|admit|l3_erase|release)|Radix|Scan' --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu2.log 2>&1
echo "launches rc=$?"
