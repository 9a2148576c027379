#!/bin/bash
# round 2f: full GPU suite (band-major long segments, device memory pool), bench, frame timeline
mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q > gpurun_out/r02f_tests.txt 2>&1
tail -3 gpurun_out/r02f_tests.txt
python bench.py --steps 20 --warmup 5 > gpurun_out/r02f_bench.json 2> gpurun_out/r02f_bench.err
python - <<'PY'
import json
d = json.loads(open("gpurun_out/r02f_bench.json").read().strip().splitlines()[-1])
print("value", d["value"], "e2e", d["e2e"]["value"], "mapping", d["mapping"]["value"], "roofline", d["roofline"]["frac"])
print("k_sweep", {k: round(v["frames_per_s"], 1) for k, v in d["k_sweep"]["k"].items()})
print("mapedit", json.dumps(d["extras"]["mapedit"]))
print("dropin", [(p["policy"], p["iterations_per_s"]) for p in d["e2e_dropin"]["policies"]])
PY
python scripts/timeline.py --mode frame --iters 4 --out gpurun_out/r02f_timeline.txt > /dev/null 2>&1; tail -25 gpurun_out/r02f_timeline.txt
