#!/bin/bash
# round 2g: chain without the zero fill, asynchronous device-mode twist, folded plan counters
mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q > gpurun_out/r02g_tests.txt 2>&1
tail -3 gpurun_out/r02g_tests.txt
python bench.py --steps 20 --warmup 5 --no-extras > gpurun_out/r02g_bench.json 2> gpurun_out/r02g_bench.err
python - <<'PY'
import json
d = json.loads(open("gpurun_out/r02g_bench.json").read().strip().splitlines()[-1])
print("value", d["value"], "ms", d["ms_per_step"], "e2e", d["e2e"]["value"], "mapping", d["mapping"]["value"])
print({k: round(v["ms_per_step"], 4) for k, v in d["phases"].items()})
PY
python scripts/timeline.py --mode frame --iters 4 --out gpurun_out/r02g_timeline.txt > /dev/null 2>&1; tail -6 gpurun_out/r02g_timeline.txt
