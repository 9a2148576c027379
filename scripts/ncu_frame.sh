# ncu --set full of the config-3 frame's main kernels (one launch each)
TAG=${1:-r02g}
ncu --set full --clock-control none --import-source on -k regex:"k_geom_fwd|k_geom_bwd|k_feat_bwd|k_gather_staged|k_pair_sum|k_project|k_materialize" -c 7 -f -o gpurun_out/${TAG}_frame python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e --no-mapping --no-extras > gpurun_out/${TAG}_ncu_frame.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_frame_launches.csv python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e --no-mapping --no-extras > /dev/null 2>&1
ls -la gpurun_out | grep $TAG
