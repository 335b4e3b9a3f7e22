python paper_2604_25899_b200/build.py > gpurun_out/build.log 2>&1
timeout 300 python -m pytest -x -q tests/test_gpu_prompts.py tests/test_gpu_batch.py 2>&1 | tail -2
timeout 300 python tools/e2e_timeline.py > gpurun_out/timeline.txt 2>&1; head -1 gpurun_out/timeline.txt
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/b3.json 2>gpurun_out/b3.err; echo bench rc=$?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_chunk_src|k_hash_staged" -c 8 --csv --log-file gpurun_out/prep_launches.csv python tools/e2e_timeline.py > gpurun_out/ncu_prep.log 2>&1; echo rc=$?
