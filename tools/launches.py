"""Summarise an ncu --metrics gpu__time_duration.sum launch list (CSV)."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[hdr]
ki, vi = h.index("Kernel Name"), h.index("Metric Value")
agg = collections.defaultdict(list)
for r in rows[hdr + 1:]:
    if len(r) > vi:
        agg[r[ki][:70]].append(float(r[vi].replace(",", "")))
ours = ("isnmf", "solve_", "fold_commit", "fresh_kernel", "stft_", "fill_")
mine = lambda k: any(x in k for x in ours)  # noqa: E731
tot = sum(sum(v) for k, v in agg.items() if mine(k))
for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
    if mine(k):
        print(f"{len(v):6d} x {sum(v) / len(v) / 1e3:9.2f} us = {sum(v) / 1e6:8.3f} ms ({100 * sum(v) / tot:5.1f}%)  {k}")
