#!/usr/bin/env python
"""Per-kernel SASS opcode mix and stall-sample share from `ncu --page source --csv`.
usage: ncu -i rep --page source --csv > src.csv; python tools/ncu_opmix.py src.csv [kernel-substring]"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
want = sys.argv[2] if len(sys.argv) > 2 else ""
blocks, cur = [], None
for r in rows:
    if r and r[0] == "Kernel Name":
        cur = {"name": r[1], "rows": []}
        blocks.append(cur)
    elif cur is not None:
        cur["rows"].append(r)
seen = set()
for b in blocks:
    if want not in b["name"] or b["name"] in seen:
        continue
    seen.add(b["name"])
    hdr = b["rows"][0]
    i_src, i_s, i_ie = hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Instructions Executed")
    ops, samp = collections.Counter(), collections.Counter()
    for r in b["rows"][1:]:
        try:
            ie, sm = float(r[i_ie] or 0), float(r[i_s] or 0)
        except (ValueError, IndexError):
            continue
        toks = r[i_src].split()
        if not toks:
            continue
        op = toks[1] if toks[0].startswith("@") else toks[0]
        op = op.split(".")[0]
        ops[op] += ie
        samp[op] += sm
    tot, ts = sum(ops.values()), sum(samp.values()) or 1
    print(f"== {b['name'][:110]}  (warp instructions {tot:.3g})")
    for op, c in ops.most_common(18):
        print(f"   {op:12s} {c / tot * 100:5.1f}% of instr   {samp[op] / ts * 100:5.1f}% of stall samples")
