# round-end refresh on a 4-GPU box: all GPU tests (multi-GPU shard tests included), smoke,
# bench at N=1 (+ reference arm), scaling N=1,2,4, launch list of the N=1 bench
python paper_2604_25899_b200/build.py > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/re_pytest.log 2>&1; tail -2 gpurun_out/re_pytest.log
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/re_bench.json 2> gpurun_out/re_bench.err; echo "bench rc=$?"
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/re_ref.json 2> gpurun_out/re_ref.err; echo "ref rc=$?"
NS="1 2 4" bash tools/gpu_scale.sh > gpurun_out/re_scale.log 2>&1; tail -4 gpurun_out/re_scale.log | cut -c1-300; cp gpurun_out/scale.jsonl gpurun_out/re_scale.jsonl
CMD="python bench.py --steps 3 --warmup 3 --profile --no-e2e --no-cpu-baseline"
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:'k_|Radix|Scan' --csv --log-file gpurun_out/re_launches.csv $CMD > gpurun_out/ncu_l.log 2>&1
echo "launches rc=$?"
