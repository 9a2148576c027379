#!/bin/bash
# round 2o: occupancy A/B of k_feat_bwd (min blocks 5 / 6) and k_geom_fwd (20 / 24 CTAs per SM)
mkdir -p gpurun_out
bash scripts/ab_libs.sh "k_feat_bwd<|k_geom_fwd" "--steps 10 --warmup 3 --no-e2e --no-mapping --no-extras --no-cpu" default fb5 fb6 fw20 fw24 default fw20 > gpurun_out/r02o_ab.txt 2>&1
cat gpurun_out/r02o_ab.txt
bash scripts/ab_libs.sh "k_geom_fwd" "--config c1 --k 16 --steps 5 --warmup 3 --no-e2e --no-mapping --no-extras --no-cpu" default fw20 >> gpurun_out/r02o_ab.txt 2>&1
tail -2 gpurun_out/r02o_ab.txt
