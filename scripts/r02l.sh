#!/bin/bash
# round 2l: branch-free generic-pointer staged gather (A/B + parity under the variant)
mkdir -p gpurun_out
export TK_RENDER_LIB=$PWD/paper_2602_06991_b200/lib/ggen/libtkrender.so
python -m pytest tests -m gpu -x -q -k "parity or fullsize or c1c2 or stress or fused" > gpurun_out/r02l_tests.txt 2>&1; tail -2 gpurun_out/r02l_tests.txt
unset TK_RENDER_LIB
bash scripts/ab_libs.sh "k_gather_staged" "--steps 10 --warmup 3 --no-e2e --no-mapping --no-extras --no-cpu" default ggen default ggen > gpurun_out/r02l_ab.txt 2>&1
cat gpurun_out/r02l_ab.txt
bash scripts/ab_libs.sh "k_gather_staged" "--config c5 --steps 5 --warmup 3 --no-e2e --no-mapping --no-extras --no-cpu" default ggen >> gpurun_out/r02l_ab.txt 2>&1
tail -2 gpurun_out/r02l_ab.txt
