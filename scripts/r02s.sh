#!/bin/bash
# round 2s: staged gather specialised for D % 512 == 0 without peers (A/B)
mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q -k "parity or fullsize or fused or c1c2 or stress" > gpurun_out/r02s_tests.txt 2>&1; tail -2 gpurun_out/r02s_tests.txt
bash scripts/ab_libs.sh "k_gather_staged" "--steps 10 --warmup 3 --no-e2e --no-mapping --no-extras --no-cpu" default nofull default nofull > gpurun_out/r02s_ab.txt 2>&1
cat gpurun_out/r02s_ab.txt
