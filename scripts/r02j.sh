#!/bin/bash
# round 2j: entry records by depth rank (materialize), items-kernel depth / occupancy A/B
mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q > gpurun_out/r02j_tests.txt 2>&1
tail -3 gpurun_out/r02j_tests.txt
bash scripts/ab_libs.sh "k_feat_bwd|k_long|k_materialize|k_sorted" "--config c1 --k 16 --steps 10 --warmup 3 --no-e2e --no-mapping --no-extras --no-cpu" \
  default it4x4 it16x2 > gpurun_out/r02j_ab.txt 2>&1
cat gpurun_out/r02j_ab.txt
for i in 1 2; do
python bench.py --steps 20 --warmup 5 --no-extras --no-e2e > gpurun_out/r02j_bench.json 2> gpurun_out/r02j_bench.err
python - <<'PY'
import json
d = json.loads(open("gpurun_out/r02j_bench.json").read().strip().splitlines()[-1])
print("value", round(d["value"], 2), "ms", round(d["ms_per_step"], 4), "mapping", round(d["mapping"]["value"], 1),
      {k: round(v["ms_per_step"], 4) for k, v in d["phases"].items()})
PY
done
