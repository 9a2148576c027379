#!/usr/bin/env python
"""Summarise an ncu launch list + an ncu --set full report into profiles/.

  python scripts/profile_summary.py TAG launches.csv report.ncu-rep [bench.json] [--title T] [--cmd C]

Writes profiles/TAG_summary.md, profiles/TAG_launches.csv and profiles/TAG_ncu_traffic.json
(DRAM bytes read+write per launch for each fully captured kernel; bench.py reads the latest
*_ncu_traffic.json to fill roofline.traffic).
"""
from __future__ import annotations

import collections
import csv
import json
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PROFILES = os.path.join(ROOT, "profiles")

WANT = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "launch__registers_per_thread", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "smsp__thread_inst_executed_per_inst_executed.ratio", "lts__throughput.avg.pct_of_peak_sustained_elapsed"]

SCALE = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ms": 1e-3, "us": 1e-6, "usecond": 1e-6,
         "msecond": 1e-3, "nsecond": 1e-9, "ns": 1e-9}


def short(name: str) -> str:
    n = name.split("(")[0].replace("(anonymous namespace)::", "").replace("void ", "")
    return n.replace("tk::", "").replace("<unnamed>::", "").replace("unnamed>::", "")


def launch_table(path: str, step_marker: str = "k_project"):
    rows = list(csv.reader(open(path)))
    hdr = [r for r in rows if "Kernel Name" in r][0]
    data = [dict(zip(hdr, r)) for r in rows if len(r) == len(hdr) and r != hdr]
    dur = [(short(d["Kernel Name"]), float(d["Metric Value"])) for d in data
           if d["Metric Name"] == "gpu__time_duration.sum"]
    starts = [i for i, (n, _) in enumerate(dur) if step_marker in n]
    last = dur[starts[-1]:] if starts else dur
    agg = collections.OrderedDict()
    for n, t in last:
        agg.setdefault(n, [0.0, 0])
        agg[n][0] += t
        agg[n][1] += 1
    return agg, sum(t for _, t in last), len(last)


def full_report(path: str):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    hdr, units, data = rows[0], rows[1], rows[2:]
    out = []
    for d in data:
        rec = {"kernel": short(d[hdr.index("Kernel Name")])}
        for w in WANT:
            if w in hdr:
                i = hdr.index(w)
                try:
                    v = float(d[i].replace(",", ""))
                except ValueError:
                    continue
                rec[w] = v * SCALE.get(units[i], 1.0) if units[i] in SCALE else v
        out.append(rec)
    return out


def main():
    argv = sys.argv[1:]
    opts = {}
    for key in ("--title", "--cmd"):
        if key in argv:
            i = argv.index(key)
            opts[key] = argv[i + 1]
            del argv[i:i + 2]
    tag, launches, rep = argv[0:3]
    bench = json.load(open(argv[3])) if len(argv) > 3 else None
    os.makedirs(PROFILES, exist_ok=True)
    shutil.copy(launches, os.path.join(PROFILES, f"{tag}_launches.csv"))
    agg, tot, n = launch_table(launches)
    title = opts.get("--title", "config 3, one bench step")
    cmd = opts.get("--cmd", "python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e")
    lines = [f"# {tag} — ncu summaries ({title})", "",
             "Launch list: `ncu --metrics gpu__time_duration.sum --clock-control none` on "
             f"`{cmd}` (cold, serialised launches: compare shares, not absolutes).", "",
             "| kernel | launches | us | share |", "|---|---|---|---|"]
    for name, (t, c) in sorted(agg.items(), key=lambda x: -x[1][0]):
        lines.append(f"| {name} | {c} | {t / 1e3:.1f} | {100 * t / tot:.1f}% |")
    lines += ["", f"Kernel time in the step: {tot / 1e3:.1f} us over {n} launches.", ""]
    recs = [r for one in rep.split(",") for r in full_report(one)]
    traffic = {}
    lines += ["## ncu --set full (per launch)", "",
              "| kernel | time ms | DRAM read GB | DRAM write GB | DRAM % | L2 % | SM % | fp64 pipe % | regs | warps active % | threads/inst |",
              "|---|---|---|---|---|---|---|---|---|---|---|"]
    seen = set()
    for r in recs:
        if r["kernel"] in seen:
            continue
        seen.add(r["kernel"])
        rd, wr = r.get("dram__bytes_read.sum", 0.0), r.get("dram__bytes_write.sum", 0.0)
        traffic[r["kernel"]] = rd + wr
        lines.append("| {} | {:.3f} | {:.3f} | {:.3f} | {:.1f} | {:.1f} | {:.1f} | {:.1f} | {:.0f} | {:.1f} | {:.1f} |".format(
            r["kernel"], r.get("gpu__time_duration.sum", 0) * 1e3, rd / 1e9, wr / 1e9,
            r.get("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", 0),
            r.get("lts__throughput.avg.pct_of_peak_sustained_elapsed", 0),
            r.get("sm__throughput.avg.pct_of_peak_sustained_elapsed", 0),
            r.get("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", 0),
            r.get("launch__registers_per_thread", 0), r.get("sm__warps_active.avg.pct_of_peak_sustained_active", 0),
            r.get("smsp__thread_inst_executed_per_inst_executed.ratio", 0)))
    if bench:
        ro = bench.get("roofline", {})
        lines += ["", "## bench line (same round)", "",
                  f"value {bench['value']:.1f} frames/s, {bench['ms_per_step']:.3f} ms/step; roofline kernel "
                  f"{ro.get('kernel')}: achieved {ro.get('achieved', 0):.0f} GB/s of {ro.get('peak')} "
                  f"({ro.get('frac', 0):.3f}); e2e {bench.get('e2e', {}).get('value')} frames/s; "
                  f"cpu_baseline {bench.get('cpu_baseline', {}).get('value')} frames/s."]
    open(os.path.join(PROFILES, f"{tag}_summary.md"), "w").write("\n".join(lines) + "\n")
    json.dump(traffic, open(os.path.join(PROFILES, f"{tag}_ncu_traffic.json"), "w"), indent=1)
    print("\n".join(lines))


if __name__ == "__main__":
    main()
