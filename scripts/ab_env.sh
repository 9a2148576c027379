#!/bin/bash
# A/B environment settings of one build on one GPU box.
#
#   bash scripts/ab_env.sh "<bench.py args>" "ENV=1 ENV2=x" "ENV=0" ...
#
# Each argument after the first is a set of VAR=value assignments (or "-" for none); bench.py runs
# once per set and its JSON line's value / e2e are printed.
set -u
bargs=$1; shift
mkdir -p gpurun_out
i=0
for envs in "$@"; do
  i=$((i+1))
  [ "$envs" = "-" ] && envs=""
  env $envs python bench.py $bargs > gpurun_out/abe_$i.json 2> gpurun_out/abe_$i.err || { echo "[$envs] failed"; tail -5 gpurun_out/abe_$i.err; continue; }
  python - "$i" "$envs" <<'PY'
import json, sys
j = json.loads(open(f"gpurun_out/abe_{sys.argv[1]}.json").read().strip().splitlines()[-1])
e2e = (j.get('e2e') or {}).get('value', float('nan'))
mp = (j.get('mapping') or {}).get('value', float('nan'))
print(f"[{sys.argv[2]}] value {j['value']:.2f} {j['unit']} ms/step {j['ms_per_step']:.3f} e2e {e2e:.3f} mapping {mp:.2f}")
PY
done
