"""Print value and per-phase ms of bench JSON lines: python scripts/show_ab.py gpurun_out/r02f_*.log"""
import json
import sys

for f in sys.argv[1:]:
    lines = [x for x in open(f) if x.startswith("{")]
    if not lines:
        print(f, "no JSON line")
        continue
    d = json.loads(lines[-1])
    ph = {k: round(v["ms_per_step"], 3) for k, v in d["phases"].items()}
    print(f"{f.split('/')[-1]:28s} {d['value']:7.1f} f/s {d['ms_per_step']:.3f} ms {ph}")
