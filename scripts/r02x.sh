#!/bin/bash
# round 2x: D % 128 staged gather / feature backward mode (config 5, D = 768) A/B; config 3 unchanged
mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q -k "stress or parity or fullsize" > gpurun_out/r02x_tests.txt 2>&1; tail -2 gpurun_out/r02x_tests.txt
bash scripts/ab_libs.sh "k_gather_staged|k_feat_bwd" "--config c5 --steps 5 --warmup 3 --no-e2e --no-mapping --no-extras --no-cpu" default prev default prev > gpurun_out/r02x_ab.txt 2>&1
bash scripts/ab_libs.sh "k_gather_staged|k_feat_bwd" "--steps 10 --warmup 3 --no-e2e --no-mapping --no-extras --no-cpu" default prev >> gpurun_out/r02x_ab.txt 2>&1
cat gpurun_out/r02x_ab.txt
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -1
