TAG=${1:-r01x}
set -x
mkdir -p gpurun_out
python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err || exit 1
python scripts/map_profile.py --iters 10 > gpurun_out/${TAG}_mp.log 2>&1 || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_frame_launches.csv python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e --no-mapping > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_geom_fwd|k_geom_bwd|k_feat_bwd|k_gather_staged|k_project|k_chain" -c 9 -f -o gpurun_out/${TAG}_frame python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e --no-mapping > gpurun_out/${TAG}_ncu_frame.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_map_launches.csv python scripts/map_profile.py --iters 10 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_feature_adam_vec|k_active_grad|k_feature_loss_staged|k_color_loss|k_ssim_stats|k_geo_adam" --launch-skip 30 -c 10 -f -o gpurun_out/${TAG}_map python scripts/map_profile.py --iters 10 > gpurun_out/${TAG}_ncu_map.log 2>&1
ls -la gpurun_out/ | grep ${TAG}
