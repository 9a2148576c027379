#!/bin/bash
# round 2k: entry records A/B (config 3 prepare), PDL / pool tests
mkdir -p gpurun_out
python -m pytest tests/test_gpu_pdl_pool.py -x -q > gpurun_out/r02k_tests.txt 2>&1; tail -3 gpurun_out/r02k_tests.txt
bash scripts/ab_libs.sh "k_materialize|k_sorted_ntiles" "--steps 10 --warmup 3 --no-e2e --no-mapping --no-extras --no-cpu" default norec default norec > gpurun_out/r02k_ab.txt 2>&1
cat gpurun_out/r02k_ab.txt
for v in default norec default norec; do
  [ $v = default ] && unset TK_RENDER_LIB || export TK_RENDER_LIB=$PWD/paper_2602_06991_b200/lib/$v/libtkrender.so
  python bench.py --steps 20 --warmup 5 --no-extras --no-e2e --no-mapping > gpurun_out/r02k_$v.json 2>/dev/null
  python -c "import json;d=json.loads(open('gpurun_out/r02k_$v.json').read().strip().splitlines()[-1]);print('$v', round(d['value'],2), {k: round(v['ms_per_step'],4) for k,v in d['phases'].items()})"
done
