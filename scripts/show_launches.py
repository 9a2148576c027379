"""Summarise an ncu --csv launch list (gpu__time_duration and optional dram bytes) per kernel."""
import collections
import csv
import sys


def main(path, top=20):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    h = rows[0]
    ki, mi, vi = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
    agg = collections.defaultdict(lambda: collections.defaultdict(float))
    cnt = collections.Counter()
    for r in rows[1:]:
        name = r[ki].split("(")[0].replace("void ", "").replace("(anonymous namespace)::", "")
        agg[name][r[mi]] += float(r[vi].replace(",", ""))
        if r[mi] == "gpu__time_duration.sum":
            cnt[name] += 1
    tot = sum(v["gpu__time_duration.sum"] for v in agg.values())
    for name, v in sorted(agg.items(), key=lambda x: -x[1]["gpu__time_duration.sum"])[:top]:
        t = v["gpu__time_duration.sum"]
        extra = " ".join(f"{m.split('__')[1].split('.')[0]}={b / 1e9:.3f}GB" for m, b in v.items() if "dram" in m)
        print(f"{name[:48]:48s} n={cnt[name]:3d} {t / 1e3:9.1f} us {100 * t / tot:5.1f}% {extra}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 20)
