# e2e check: prompts/pipeline GPU tests, then the default bench line (+ e2e) and the breakdown tool
python paper_2604_25899_b200/build.py > gpurun_out/build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_prompts.py -x -q 2>&1 | tail -2
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline ${BENCH_ARGS} > gpurun_out/e2e.json 2> gpurun_out/e2e.err; echo "bench rc=$?"
timeout 300 python tools/e2e_breakdown.py > gpurun_out/breakdown.txt 2>&1; cat gpurun_out/breakdown.txt | tail -2
