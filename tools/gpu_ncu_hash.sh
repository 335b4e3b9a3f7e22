set -x
python paper_2604_25899_b200/build.py > gpurun_out/build.log 2>&1
CMD="python bench.py --steps 2 --warmup 1 --workflows 3000 --no-e2e --no-cpu-baseline"
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_hash_staged -s 1 -c 1 -o gpurun_out/prof_hash $CMD > gpurun_out/ncu.log 2>&1
echo "ncu rc=$?"
tail -3 gpurun_out/ncu.log
$CMD > gpurun_out/plain2.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu2.log 2>&1
echo "ncu2 rc=$?"
