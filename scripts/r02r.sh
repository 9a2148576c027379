#!/bin/bash
# round 2r: K <= 3 staged gather / feature loss instantiated at KMAX = 3 (A/B against KMAX = 4)
mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q -k "parity or fullsize or mapping or lazy or fused" > gpurun_out/r02r_tests.txt 2>&1; tail -2 gpurun_out/r02r_tests.txt
bash scripts/ab_libs.sh "k_gather_staged|k_feature_loss" "--steps 10 --warmup 3 --no-e2e --no-extras --no-cpu" default k4 default k4 > gpurun_out/r02r_ab.txt 2>&1
cat gpurun_out/r02r_ab.txt
