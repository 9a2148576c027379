#!/bin/bash
# round 2v: feature backward fast path for all-finite record batches (A/B)
mkdir -p gpurun_out
TK_RENDER_LIB=$PWD/paper_2602_06991_b200/lib/ff/libtkrender.so python -m pytest tests -m gpu -x -q -k "parity or fullsize or c1c2 or long or async" > gpurun_out/r02v_tests.txt 2>&1; tail -2 gpurun_out/r02v_tests.txt
bash scripts/ab_libs.sh "k_feat_bwd" "--steps 10 --warmup 3 --no-e2e --no-mapping --no-extras --no-cpu" default ff default ff > gpurun_out/r02v_ab.txt 2>&1
bash scripts/ab_libs.sh "k_feat_bwd" "--config c1 --k 16 --steps 5 --warmup 3 --no-e2e --no-mapping --no-extras --no-cpu" default ff >> gpurun_out/r02v_ab.txt 2>&1
cat gpurun_out/r02v_ab.txt
