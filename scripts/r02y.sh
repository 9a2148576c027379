#!/bin/bash
# round 2y: geometry-backward merge with grouped partial loads (A/B)
mkdir -p gpurun_out
bash scripts/ab_libs.sh "k_mid_small" "--steps 10 --warmup 3 --no-e2e --no-mapping --no-extras --no-cpu" default mg2 mg4 default mg2 mg4 > gpurun_out/r02y_ab.txt 2>&1
cat gpurun_out/r02y_ab.txt
TK_RENDER_LIB=$PWD/paper_2602_06991_b200/lib/mg2/libtkrender.so python -m pytest tests -m gpu -x -q -k "fullsize or c1c2 or parity" > gpurun_out/r02y_tests.txt 2>&1; tail -1 gpurun_out/r02y_tests.txt
