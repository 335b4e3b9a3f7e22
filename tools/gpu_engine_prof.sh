#!/bin/bash
# engine_b200 call profile at WF workflows (PYG_ADAPTER_PROFILE) + K1 sweep
set -x
python paper_2604_25899_b200/build.py > gpurun_out/build.log 2>&1
mkdir -p gpurun_out/ep
t0=$(date +%s%N); PYG_ADAPTER_PROFILE=1 PYG_ENGINE_MAX_REPLICAS=1024 ./integration/_build/engine_b200 gpurun_out/ep ${WF:-200} 1 > gpurun_out/engine_prof.txt 2>&1; echo "b200 wall_ms $(( ($(date +%s%N) - t0) / 1000000 ))" >> gpurun_out/engine_prof.txt
rm -rf gpurun_out/ep
head -30 gpurun_out/engine_prof.txt
timeout 600 python tools/k1_sweep.py > gpurun_out/k1_sweep.jsonl 2>&1; cat gpurun_out/k1_sweep.jsonl
