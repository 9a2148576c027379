#!/bin/bash
# round-2 final mapping-step profile (config 3, tk_optimize_step, feature steps every 5th iteration)
mkdir -p gpurun_out
python scripts/map_profile.py --iters 10 > gpurun_out/r02e_mp.log 2>&1 &&
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02e_map_launches.csv python scripts/map_profile.py --iters 10 > /dev/null 2>&1 &&
ncu --set full --clock-control none --import-source on -k regex:"k_feature_adam_vec|k_active_grad|k_feature_loss_staged|k_color_loss|k_ssim_stats|k_geo_adam" --launch-skip 30 -c 10 -f -o gpurun_out/r02e_map python scripts/map_profile.py --iters 10 > gpurun_out/r02e_ncu_map.log 2>&1
tail -5 gpurun_out/r02e_mp.log; ls -la gpurun_out | grep r02e_map
