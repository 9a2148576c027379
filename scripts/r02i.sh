#!/bin/bash
# round 2h: selective PDL (prepare and index chains), chain reverted to zero fill + rank chain
mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q > gpurun_out/r02i_tests.txt 2>&1
tail -3 gpurun_out/r02i_tests.txt
for pdl in 1 0 1 0; do
  TK_PDL=$pdl python bench.py --steps 20 --warmup 5 --no-extras --no-e2e > gpurun_out/r02i_bench_$pdl.json 2> gpurun_out/r02i_bench_$pdl.err
  python - $pdl <<'PY'
import json, sys
d = json.loads(open(f"gpurun_out/r02i_bench_{sys.argv[1]}.json").read().strip().splitlines()[-1])
print("PDL", sys.argv[1], "value", round(d["value"], 2), "ms", round(d["ms_per_step"], 4), "mapping", round(d["mapping"]["value"], 1),
      {k: round(v["ms_per_step"], 4) for k, v in d["phases"].items()})
PY
done
python scripts/timeline.py --mode frame --iters 4 --out gpurun_out/r02i_timeline.txt > /dev/null 2>&1; tail -4 gpurun_out/r02i_timeline.txt
TK_PDL=0 python scripts/timeline.py --mode frame --iters 4 --out gpurun_out/r02i_timeline0.txt > /dev/null 2>&1; tail -4 gpurun_out/r02i_timeline0.txt
