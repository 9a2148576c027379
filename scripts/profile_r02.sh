# round-2 profile set: frame launch list + ncu --set full of the frame kernels + bench line
TAG=${1:-r02}
A="--steps 1 --warmup 3 --no-cpu --no-e2e --no-mapping --no-extras"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_frame_launches.csv python bench.py $A > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_project|k_materialize|k_geom_fwd|k_gather_staged|k_feat_bwd<|k_geom_bwd|k_mid_small|k_chain|k_slot_keys|k_rs_scatter" -c 14 -f -o gpurun_out/${TAG}_frame python bench.py $A > gpurun_out/${TAG}_ncu_frame.log 2>&1
ls -la gpurun_out | grep $TAG
