#!/bin/bash
# round 2t: feature backward and feature loss specialised for D % 512 == 0 (A/B), tests
mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q -k "parity or fullsize or mapping or lazy or c1c2 or long" > gpurun_out/r02t_tests.txt 2>&1; tail -2 gpurun_out/r02t_tests.txt
bash scripts/ab_libs.sh "k_feat_bwd|k_feature_loss" "--steps 10 --warmup 3 --no-e2e --no-extras --no-cpu" default base default base > gpurun_out/r02t_ab.txt 2>&1
cat gpurun_out/r02t_ab.txt
