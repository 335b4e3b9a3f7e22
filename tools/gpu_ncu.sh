# usage: KERNEL=k_hash_staged bash tools/gpu_ncu.sh   (profiles one launch of KERNEL at full scale)
set -x
python paper_2604_25899_b200/build.py > gpurun_out/build.log 2>&1
CMD="python bench.py --steps 3 --warmup 1 --profile --no-e2e --no-cpu-baseline"
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:${KERNEL} -s 1 -c 1 -o gpurun_out/prof_${KERNEL} $CMD > gpurun_out/ncu_${KERNEL}.log 2>&1
echo "ncu rc=$?"
tail -2 gpurun_out/ncu_${KERNEL}.log
if [ -n "$LAUNCHES" ]; then
$CMD > gpurun_out/plain2.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:'k_|Radix|Scan' --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu2.log 2>&1
echo "launches rc=$?"
fi
