"""Summarise an ncu --metrics gpu__time_duration.sum launch list (second query only)."""
import csv
import sys
from collections import defaultdict


def load(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hi]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    return [(r[ki].split("(")[0].replace("void ", ""), float(r[vi].replace(",", ""))) for r in rows[hi + 1:]]


def main(path, queries=2):
    seq = load(path)
    per_q = len(seq) // queries
    last = seq[-per_q:]
    tot = defaultdict(float)
    cnt = defaultdict(int)
    for name, ns in last:
        base = name.split("<")[0]
        tot[base] += ns
        cnt[base] += 1
    allns = sum(tot.values())
    print(f"{path}: {len(last)} launches, {allns/1e3:.1f} us (ncu, serialised, cold L2)")
    for k in sorted(tot, key=lambda x: -tot[x]):
        print(f"  {k:16s} n={cnt[k]:3d}  {tot[k]/1e3:9.1f} us  {100*tot[k]/allns:5.1f}%")


if __name__ == "__main__":
    for p in sys.argv[1:]:
        main(p)
