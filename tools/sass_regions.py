"""Per-region breakdown of an ncu source (SASS) export: samples, stall reasons and
instruction mix between consecutive barriers.  usage: sass_regions.py sass.csv"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr, data = rows[1], rows[2:]
col = {n: i for i, n in enumerate(hdr)}


def I(x):
    try:
        return int(x)
    except ValueError:
        return 0


stalls = [n for n in hdr if n.startswith("stall_") and "Not Issued" not in n]
seg, cur = [], None
for i, r in enumerate(data):
    if cur is None:
        cur = {"lo": i, "samples": 0, "hmma": 0, "inst": 0, "st": collections.Counter(), "ops": collections.Counter()}
    ins = r[1].strip()
    cur["samples"] += I(r[col["# Samples"]])
    ex = I(r[col["Instructions Executed"]])
    op = (ins.split()[1] if ins.startswith("@") else ins.split()[0]).split(".")[0]
    cur["ops"][op] += ex
    cur["inst"] += ex
    for s in stalls:
        cur["st"][s[6:]] += I(r[col[s]])
    if "BAR.SYNC" in ins or "EXIT" in ins or "BAR.RED" in ins:
        cur["hi"] = i
        seg.append(cur)
        cur = None
tot = sum(s["samples"] for s in seg) or 1
for s in seg:
    if s["samples"] < 0.01 * tot:
        continue
    print(f"insts {s['lo']:5d}-{s['hi']:5d}: {100 * s['samples'] / tot:5.1f}% of samples, HMMA {s['ops']['HMMA']}, "
          f"instructions {s['inst']}")
    print("   stalls:", ", ".join(f"{k} {v}" for k, v in s["st"].most_common(6)))
    print("   ops:   ", ", ".join(f"{k} {v}" for k, v in s["ops"].most_common(8)))
