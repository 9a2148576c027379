#!/bin/bash
# round 2n: k_chain occupancy A/B (config 3)
mkdir -p gpurun_out
bash scripts/ab_libs.sh "k_chain" "--steps 10 --warmup 3 --no-e2e --no-mapping --no-extras --no-cpu" default ch4 ch6 default ch4 > gpurun_out/r02n_ab.txt 2>&1
cat gpurun_out/r02n_ab.txt
python -m pytest tests/test_gpu_pdl_pool.py -x -q 2>&1 | tail -1
