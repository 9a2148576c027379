#!/bin/bash
# round 2u: staged gather with all record rows of a channel quad loaded before the FMAs (A/B)
mkdir -p gpurun_out
TK_RENDER_LIB=$PWD/paper_2602_06991_b200/lib/pq/libtkrender.so python -m pytest tests -m gpu -x -q -k "parity or fullsize" > gpurun_out/r02u_tests.txt 2>&1; tail -2 gpurun_out/r02u_tests.txt
bash scripts/ab_libs.sh "k_gather_staged" "--steps 10 --warmup 3 --no-e2e --no-mapping --no-extras --no-cpu" default pq default pq > gpurun_out/r02u_ab.txt 2>&1
bash scripts/ab_libs.sh "k_gather_staged" "--config c5 --steps 5 --warmup 3 --no-e2e --no-mapping --no-extras --no-cpu" default pq >> gpurun_out/r02u_ab.txt 2>&1
cat gpurun_out/r02u_ab.txt
