"""Aggregate an ncu --metrics gpu__time_duration.sum CSV launch list into
per-kernel totals and shares.  python tools/launch_share.py launches.csv [skip_first_n]"""
import csv
import sys
from collections import defaultdict

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
hdr = rows[0]
ik, iv, im = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Name")
skip = int(sys.argv[2]) if len(sys.argv) > 2 else 0
tot = defaultdict(float)
cnt = defaultdict(int)
for r in rows[1 + skip:]:
    if r[im] != "gpu__time_duration.sum":
        continue
    name = r[ik].split("(")[0][:80]
    tot[name] += float(r[iv].replace(",", ""))
    cnt[name] += 1
allt = sum(tot.values())
print(f"total {allt / 1e3:.1f} us over {sum(cnt.values())} launches")
for k, v in sorted(tot.items(), key=lambda kv: -kv[1]):
    print(f"{v / allt * 100:6.2f}%  {v / 1e3:9.1f} us  x{cnt[k]:4d}  {k}")
