# usage: TESTS="tests/test_x.py" BENCH_ARGS="..." bash tools/gpu_quick.sh
set -x
python paper_2604_25899_b200/build.py > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest ${TESTS:-tests} -x -q -m gpu 2>&1 | tail -25
if [ -n "$BENCH" ]; then
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline ${BENCH_ARGS} > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
tail -5 gpurun_out/bench.err
cat gpurun_out/bench.json
fi
