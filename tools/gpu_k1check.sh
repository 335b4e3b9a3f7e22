#!/bin/bash
python paper_2604_25899_b200/build.py > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
timeout 600 python -m pytest -q -m gpu tests/test_gpu_batch.py -k hash 2>&1 | tail -1
python tools/k1_sweep.py --sizes 16000,125000 --splits=-1,10240 --grids persistent | cut -c1-100
GRIDS="${GRIDS:-persistent tasks}" bash tools/gpu_quick_ab.sh
