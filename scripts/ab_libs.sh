#!/bin/bash
# A/B alternative builds of libtkrender.so on one GPU box.
#
#   bash scripts/ab_libs.sh "<ncu kernel regex>" "<bench.py args>" default varA varB ...
#
# "default" is paper_2602_06991_b200/lib/libtkrender.so; any other name is
# paper_2602_06991_b200/lib/<name>/libtkrender.so (loaded through TK_RENDER_LIB).  Each variant
# runs bench.py once without ncu (its JSON line), then once under an ncu launch list of the
# kernels matching the regex; prints the median launch time per kernel and the bench values.
set -u
regex=$1; bargs=$2; shift 2
mkdir -p gpurun_out
for v in "$@"; do
  if [ "$v" = default ]; then unset TK_RENDER_LIB; else export TK_RENDER_LIB=$PWD/paper_2602_06991_b200/lib/$v/libtkrender.so; fi
  python bench.py $bargs > gpurun_out/ab_$v.json 2> gpurun_out/ab_$v.err || { echo "$v failed"; tail -5 gpurun_out/ab_$v.err; continue; }
  ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"$regex" --csv \
      --log-file gpurun_out/ab_$v.csv python bench.py $bargs > /dev/null 2>&1
  python - "$v" <<'PY'
import csv, json, statistics, sys
v = sys.argv[1]
rows = [r for r in csv.reader(open(f"gpurun_out/ab_{v}.csv")) if len(r) > 10]
h = rows[0]
by = {}
for r in rows[1:]:
    by.setdefault(r[h.index("Kernel Name")].split("(")[0][-40:], []).append(float(r[h.index("Metric Value")]))
j = json.loads(open(f"gpurun_out/ab_{v}.json").read().strip().splitlines()[-1])
ker = ", ".join(f"{k} {statistics.median(t) / 1e3:.1f}us x{len(t)}" for k, t in sorted(by.items()))
e2e = (j.get("e2e") or {}).get("value", float("nan"))
map_v = (j.get("mapping") or {}).get("value", float("nan"))
print(f"{v}: value {j['value']:.2f} e2e {e2e:.3f} mapping {map_v:.2f} | {ker}")
PY
done
