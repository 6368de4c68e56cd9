#!/usr/bin/env python
"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list into markdown.
usage: python tools/launch_summary.py gpurun_out/launches.csv profiles/rNN_launches.md "<command>" """
import collections
import csv
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
hdr = rows[0]
ix = {h: i for i, h in enumerate(hdr)}
agg = collections.OrderedDict()
for r in rows[1:]:
    if r[ix["Metric Name"]] != "gpu__time_duration.sum":
        continue
    name = r[ix["Kernel Name"]]
    unit = r[ix["Metric Unit"]]
    v = float(r[ix["Metric Value"]].replace(",", ""))
    ms = v / 1e6 if unit in ("nsecond", "ns") else (v / 1e3 if unit in ("usecond", "us") else v)
    n, t = agg.get(name, (0, 0.0))
    agg[name] = (n + 1, t + ms)
ours = sum(t for k, (n, t) in agg.items() if "hb::" in k)
lines = [f"# Launch list of `{sys.argv[3]}` under ncu", "",
         "`ncu --metrics gpu__time_duration.sum --clock-control none` (cold, serialised replays: "
         "compare shares, not absolutes).", "",
         "| kernel | launches | total ms | share of our kernels |", "|---|---|---|---|"]
for k, (n, t) in agg.items():
    share = f"{100 * t / ours:.1f}%" if "hb::" in k else "(torch: input generation / copies)"
    lines.append(f"| `{k[:90]}` | {n} | {t:.3f} | {share} |")
open(sys.argv[2], "w").write("\n".join(lines) + "\n")
print("\n".join(lines))
