# K1/step overlap sweep: bench.py --free-sms F for each F in $FREE (default "-1 0 8 16")
python paper_2604_25899_b200/build.py > gpurun_out/build.log 2>&1
for f in ${FREE:--1 0 8 16}; do
  timeout 300 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --free-sms $f ${BENCH_ARGS} > gpurun_out/ov_$f.json 2> gpurun_out/ov_$f.err; echo "free=$f rc=$?"
done
