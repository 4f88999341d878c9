"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list:
mean duration of each kernel over its last N launches (the timed steps)."""
import collections
import csv
import sys


def summary(path, last=3):
    lines = [l for l in open(path) if l.startswith('"')]
    rows = list(csv.reader(lines))
    h = rows[0]
    ik, iv = h.index("Kernel Name"), h.index("Metric Value")
    d = collections.defaultdict(list)
    for r in rows[1:]:
        d[r[ik].split("(")[0].replace("void ", "")[:70]].append(float(r[iv].replace(",", "")) / 1000.0)
    return {k: (len(v), sum(v[-last:]) / len(v[-last:])) for k, v in d.items()}


if __name__ == "__main__":
    last = int(sys.argv[2]) if len(sys.argv) > 2 else 3
    s = summary(sys.argv[1], last)
    for k, (n, us) in sorted(s.items(), key=lambda x: -x[1][1]):
        print(f"{k:70s} n={n:5d} mean(last {last}) {us:9.2f} us")
