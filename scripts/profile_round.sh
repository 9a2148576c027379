set -x
mkdir -p gpurun_out
python bench.py > gpurun_out/r01e_bench.json 2> gpurun_out/r01e_bench.err || exit 1
python scripts/map_profile.py --iters 10 > gpurun_out/r01e_mp.log 2>&1 || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r01e_frame_launches.csv python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e --no-mapping > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_geom_fwd|k_geom_bwd|k_feat_bwd<|k_gather_staged|k_project|k_chain" -c 6 -f -o gpurun_out/r01e_frame python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e --no-mapping > gpurun_out/r01e_ncu_frame.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r01e_map_launches.csv python scripts/map_profile.py --iters 10 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_feature_adam_vec|k_feature_loss_vec|k_color_loss|k_ssim_stats|k_geo_adam|k_topk_stats|k_rs_scatter" --launch-skip 40 -c 8 -f -o gpurun_out/r01e_map python scripts/map_profile.py --iters 10 > gpurun_out/r01e_ncu_map.log 2>&1
ls -la gpurun_out/ | grep r01e
