#!/bin/bash
# round-2 final profile set: config-3 frame launch list + ncu --set full of the four big kernels,
# config-1 K=16 feature backward (band-major long items) launch list + ncu --set full
mkdir -p gpurun_out
A="--steps 1 --warmup 3 --no-cpu --no-e2e --no-mapping --no-extras"
B="--config c1 --k 16 --steps 1 --warmup 3 --no-cpu --no-e2e --no-mapping --no-extras"
python bench.py $A > gpurun_out/r02e_plain_a.log 2>&1 &&
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02e_frame_launches.csv python bench.py $A > /dev/null 2>&1 &&
ncu --set full --clock-control none --import-source on -k regex:"k_geom_fwd|k_gather_staged|k_feat_bwd|k_geom_bwd|k_project|k_materialize|k_mid_small|k_chain" -c 12 -f -o gpurun_out/r02e_frame python bench.py $A > gpurun_out/r02e_ncu_frame.log 2>&1
python bench.py $B > gpurun_out/r02e_plain_b.log 2>&1 &&
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02e_k16_launches.csv python bench.py $B > /dev/null 2>&1 &&
ncu --set full --clock-control none -k regex:"k_feat_bwd|k_long_combine|k_gather_staged" -c 5 -f -o gpurun_out/r02e_k16 python bench.py $B > gpurun_out/r02e_ncu_k16.log 2>&1
ls -la gpurun_out | grep r02e_
