# round-end evidence: GPU tests, smoke, bench (+reference arm), launch list, K1 ncu capture
python paper_2604_25899_b200/build.py > gpurun_out/build.log 2>&1
timeout 1200 python -m pytest tests -x -q -m gpu > gpurun_out/final_pytest.log 2>&1; tail -2 gpurun_out/final_pytest.log
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/final_bench.json 2> gpurun_out/final_bench.err; echo "bench rc=$?"
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/final_ref.json 2> gpurun_out/final_ref.err; echo "ref rc=$?"
CMD="python bench.py --steps 3 --warmup 3 --profile --no-e2e --no-cpu-baseline"
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:'k_|Radix|Scan' --csv --log-file gpurun_out/final_launches.csv $CMD > gpurun_out/ncu_l.log 2>&1
echo "launches rc=$?"
ncu --set full --clock-control none --import-source on -k regex:k_hash_staged -s 3 -c 1 -o gpurun_out/final_k1 $CMD > gpurun_out/ncu_k1.log 2>&1
echo "k1 ncu rc=$?"
ncu --set full --clock-control none --import-source on -k regex:k_route_seq -s 3 -c 1 -o gpurun_out/final_k3 $CMD > gpurun_out/ncu_k3.log 2>&1
echo "k3 ncu rc=$?"
