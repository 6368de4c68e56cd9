#!/usr/bin/env python
"""Stall samples per (opcode, reason) from `ncu --page source --csv` (SASS view).
usage: python tools/ncu_stalls_by_op.py src.csv [kernel-substring] [top]"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
want = sys.argv[2] if len(sys.argv) > 2 else ""
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
blocks, cur = [], None
for r in rows:
    if r and r[0] == "Kernel Name":
        cur = {"name": r[1], "rows": []}
        blocks.append(cur)
    elif cur is not None:
        cur["rows"].append(r)
for b in blocks:
    if want not in b["name"]:
        continue
    hdr = b["rows"][0]
    i_src = hdr.index("Source")
    reasons = [(i, h) for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
    agg = collections.Counter()
    tot = 0.0
    for r in b["rows"][1:]:
        toks = r[i_src].split() if len(r) > i_src else []
        if not toks:
            continue
        op = (toks[1] if toks[0].startswith("@") else toks[0]).split(".")[0]
        for i, h in reasons:
            try:
                v = float(r[i] or 0)
            except ValueError:
                continue
            agg[(op, h[6:])] += v
            tot += v
    print(f"== {b['name'][:100]}")
    for (op, h), v in agg.most_common(top):
        print(f"   {op:10s} {h:18s} {100 * v / tot:5.1f}%")
    break
