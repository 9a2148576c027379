#!/bin/bash
# round 2aa: k_active_grad specialised for D % 512 == 0 (A/B on the mapping step), full GPU tests
mkdir -p gpurun_out
bash scripts/ab_libs.sh "k_active_grad" "--steps 20 --warmup 5 --no-e2e --no-extras --no-cpu" default base default base > gpurun_out/r02aa_ab.txt 2>&1
cat gpurun_out/r02aa_ab.txt
python -m pytest tests -m gpu -x -q > gpurun_out/r02aa_tests.txt 2>&1; tail -2 gpurun_out/r02aa_tests.txt
