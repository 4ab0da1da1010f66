"""Kernel shares of an ncu launch list (``--metrics gpu__time_duration.sum --csv``):

    python tools/ncu_launch_summary.py gpurun_out/ncu_r02/launches_default_bench.csv
"""
import collections
import csv
import sys

rows = [r for r in csv.reader(l for l in open(sys.argv[1]) if l.startswith('"'))]
h = rows[0]
ik, iv, iu = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
tot = collections.defaultdict(float)
cnt = collections.Counter()
for r in rows[1:]:
    v = float(r[iv].replace(",", ""))
    us = v / 1e3 if r[iu].startswith("ns") else v * 1e3 if r[iu].startswith("ms") else v
    tot[r[ik]] += us
    cnt[r[ik]] += 1
allus = sum(tot.values())
print("gpu__time_duration.sum by kernel over the default bench command (ncu launch list, cold-cache serialised launches)")
for k, v in sorted(tot.items(), key=lambda kv: -kv[1]):
    print(f"{100 * v / allus:6.2f}%  {v:12.1f} us  x{cnt[k]:<3d} {k[:70]}")
