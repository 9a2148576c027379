# round-2 second capture: the kernels the first one missed (feature backward, merge, chain, index)
TAG=${1:-r02b}
A="--steps 1 --warmup 3 --no-cpu --no-e2e --no-mapping --no-extras"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_frame_launches.csv python bench.py $A > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_feat_bwd<|k_geom_bwd|k_mid_small|k_mid_big|k_chain|k_slot_keys|k_gather_staged" -c 7 -f -o gpurun_out/${TAG}_frame python bench.py $A > gpurun_out/${TAG}_ncu_frame.log 2>&1
ls -la gpurun_out | grep $TAG
