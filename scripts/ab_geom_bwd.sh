set -x
python bench.py --steps 10 --warmup 3 --no-e2e --no-mapping --no-extras --no-cpu > gpurun_out/r02c_det.log 2>&1
TK_GEOM_BWD_ATOMIC=1 python bench.py --steps 10 --warmup 3 --no-e2e --no-mapping --no-extras --no-cpu > gpurun_out/r02c_atomic.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_geom_bwd|k_mid_|k_pair_sum|k_chain|k_geom_fwd" -c 40 --csv --log-file gpurun_out/r02c_launches.csv python bench.py --steps 3 --warmup 3 --no-e2e --no-mapping --no-extras --no-cpu > /dev/null 2>&1
echo done
