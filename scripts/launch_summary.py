"""Summarise an ncu --metrics gpu__time_duration.sum launch list (CSV log) per kernel.
usage: python scripts/launch_summary.py launches.csv "<command it profiled>" > summary.txt"""
import csv, sys
from collections import defaultdict
rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 5]
hdr = rows[0]
ik, im, iv = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
tot, cnt = defaultdict(float), defaultdict(int)
unit = rows[1][hdr.index("Metric Unit")] if len(rows) > 1 else "ns"
scale = {"ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0, "nsecond": 1e-6}.get(unit, 1e-6)
for r in rows[1:]:
    if r[im] != "gpu__time_duration.sum":
        continue
    tot[r[ik]] += float(r[iv].replace(",", "")) * scale
    cnt[r[ik]] += 1
share_total = sum(v for k, v in tot.items() if "gen_kernel" not in k)
print(f"# ncu launch list (gpu__time_duration.sum, --clock-control none) of: {sys.argv[2] if len(sys.argv) > 2 else ''}")
print("# (cold-cache, serialised per launch; compare SHARES). gen_kernel is the untimed input generator, excluded from the share.")
print(f"{'total_ms':>10s}  share% launches  kernel")
for k, v in sorted(tot.items(), key=lambda x: -x[1]):
    sh = "" if "gen_kernel" in k else f"{100 * v / share_total:6.2f}"
    print(f"{v:10.3f}  {sh:>6s} {cnt[k]:8d}  {k[:90]}")
