#!/bin/bash
# round 2m: pixel-ordered feature backward for K >= 8 (A/B via TK_FBWD_ORDER), tests
mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q -k "pdl or c1c2 or long or parity" > gpurun_out/r02m_tests.txt 2>&1; tail -2 gpurun_out/r02m_tests.txt
A="--config c1 --k 16 --steps 10 --warmup 3 --no-e2e --no-mapping --no-extras --no-cpu"
for o in 1 0 1 0; do
  TK_FBWD_ORDER=$o python bench.py $A > gpurun_out/r02m_$o.json 2>/dev/null
  python -c "import json;d=json.loads(open('gpurun_out/r02m_$o.json').read().strip().splitlines()[-1]);print('order $o K16', round(d['value'],2), {k: round(v['ms_per_step'],4) for k,v in d['phases'].items()})"
done
for o in 1 0; do
  TK_FBWD_ORDER=$o python bench.py --config c1 --k 8 --steps 10 --warmup 3 --no-e2e --no-mapping --no-extras --no-cpu > gpurun_out/r02m_k8_$o.json 2>/dev/null
  python -c "import json;d=json.loads(open('gpurun_out/r02m_k8_$o.json').read().strip().splitlines()[-1]);print('order $o K8', round(d['value'],2), {k: round(v['ms_per_step'],4) for k,v in d['phases'].items()})"
  TK_FBWD_ORDER=$o python bench.py --steps 10 --warmup 3 --no-e2e --no-mapping --no-extras --no-cpu > gpurun_out/r02m_c3_$o.json 2>/dev/null
  python -c "import json;d=json.loads(open('gpurun_out/r02m_c3_$o.json').read().strip().splitlines()[-1]);print('order $o c3', round(d['value'],2), {k: round(v['ms_per_step'],4) for k,v in d['phases'].items()})"
done
