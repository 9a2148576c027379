# ncu --set full of one kernel of the config-3 frame: bash scripts/ncu_one.sh TAG REGEX [extra bench args]
TAG=$1; RE=$2; shift 2
ncu --set full --clock-control none --import-source on -k regex:"$RE" -c 1 -f -o gpurun_out/${TAG} python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e --no-mapping --no-extras "$@" > gpurun_out/${TAG}.log 2>&1
ls -la gpurun_out | grep $TAG
