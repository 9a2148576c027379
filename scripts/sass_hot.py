"""Opcode mix and hot regions of one kernel's SASS from an ncu report (source page):
  python scripts/sass_hot.py report.ncu-rep KERNEL_REGEX [min_count]"""
import collections
import csv
import io
import subprocess
import sys


def main(rep, regex, minc=0):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", f"regex:{regex}",
                          "--print-source", "sass"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h = rows[1]
    data = [r for r in rows[2:] if len(r) == len(h)]  # one kernel's rows (a report may hold several)
    si, ie = h.index("Source"), h.index("Instructions Executed")
    ws = h.index("Warp Stall Sampling (All Samples)")
    vals = [int(r[ie]) if r[ie].isdigit() else 0 for r in data]
    samp = [int(r[ws]) if r[ws].isdigit() else 0 for r in data]
    tot, tots = sum(vals), max(1, sum(samp))
    op, st = collections.Counter(), collections.Counter()
    for r, v, sm in zip(data, vals, samp):
        toks = r[si].split()
        if not toks:
            continue
        o = (toks[1] if toks[0].startswith("@") else toks[0]).split(".")[0]
        op[o] += v
        st[o] += sm
    print(f"instructions {tot}  samples {tots}")
    for o, c in op.most_common(22):
        print(f"  {o:10s} {100 * c / tot:5.1f}% inst {100 * st[o] / tots:5.1f}% samples")
    if minc:
        for i, (r, v) in enumerate(zip(data, vals)):
            if v >= minc:
                print(f"{i:5d} {v / 1e3:8.0f}K {samp[i]:5d}  {r[si][:96]}")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], int(sys.argv[3]) if len(sys.argv) > 3 else 0)
