# per-phase times and the ncu launch list of the config-2 frame at large K
for k in 8 16; do
  python bench.py --config c1 --k $k --steps 5 --warmup 3 --no-e2e --no-mapping --no-extras --no-cpu > gpurun_out/r02e_k$k.log 2>&1
done
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 80 --csv --log-file gpurun_out/r02e_k16_launches.csv python bench.py --config c1 --k 16 --steps 1 --warmup 3 --no-e2e --no-mapping --no-extras --no-cpu > /dev/null 2>&1
echo done
