"""Summarise an ncu --metrics gpu__time_duration.sum launch list (CSV) into
per-kernel totals and shares. Usage: python summarize_launches.py launches.csv"""
import csv
import re
import sys
from collections import defaultdict


def main(path):
    rows = list(csv.reader(open(path)))
    hdr = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    cols = rows[hdr]
    ki, vi = cols.index("Kernel Name"), cols.index("Metric Value")
    tot = defaultdict(float)
    cnt = defaultdict(int)
    for r in rows[hdr + 1:]:
        if len(r) <= vi:
            continue
        name = re.sub(r"\(.*", "", r[ki]).replace("void ", "")
        tot[name] += float(r[vi].replace(",", "")) / 1e6
        cnt[name] += 1
    s = sum(tot.values())
    print(f"{'kernel':40s} {'launches':>8s} {'total ms':>10s} {'avg ms':>9s} {'share':>7s}")
    for k, v in sorted(tot.items(), key=lambda kv: -kv[1]):
        print(f"{k:40s} {cnt[k]:8d} {v:10.3f} {v / cnt[k]:9.4f} {100 * v / s:6.1f}%")
    print(f"{'TOTAL':40s} {sum(cnt.values()):8d} {s:10.3f}")


if __name__ == "__main__":
    main(sys.argv[1])
