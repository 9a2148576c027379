#!/bin/bash
# round 2p: k_feat_bwd at 5 resident blocks (48 registers) against the default 64-register build
mkdir -p gpurun_out
bash scripts/ab_libs.sh "k_feat_bwd" "--steps 10 --warmup 3 --no-e2e --no-mapping --no-extras --no-cpu" default fb5 default fb5 > gpurun_out/r02p_ab.txt 2>&1
cat gpurun_out/r02p_ab.txt
for v in default fb5; do
  [ $v = default ] && unset TK_RENDER_LIB || export TK_RENDER_LIB=$PWD/paper_2602_06991_b200/lib/$v/libtkrender.so
  python bench.py --steps 20 --warmup 5 --no-extras --no-e2e --no-cpu > gpurun_out/r02p_$v.json 2>/dev/null
  python -c "import json;d=json.loads(open('gpurun_out/r02p_$v.json').read().strip().splitlines()[-1]);print('$v', round(d['value'],2), 'map', round(d['mapping']['value'],1), {k: round(v['ms_per_step'],4) for k,v in d['phases'].items()})"
done
