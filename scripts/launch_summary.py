"""Per-kernel shares of an ncu launch list (--metrics gpu__time_duration.sum
--csv): python scripts/launch_summary.py launches.csv [out.txt]"""
import csv
import re
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[hi]
ki, mi, vi = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
unit_i = h.index("Metric Unit") if "Metric Unit" in h else None
tot = defaultdict(float)
cnt = defaultdict(int)
for r in rows[hi + 1:]:
    if len(r) <= vi or r[mi] != "gpu__time_duration.sum":
        continue
    v = float(r[vi].replace(",", ""))
    u = r[unit_i] if unit_i is not None else "ns"
    v_us = v / 1000.0 if u in ("ns", "nsecond") else v * (1000.0 if u in ("ms", "msecond") else 1.0)
    name = re.sub(r"\(.*", "", r[ki]).replace("void ", "").strip()
    tot[name] += v_us
    cnt[name] += 1
T = sum(tot.values())
lines = [f"{'kernel':60s} {'launches':>8s} {'total ms':>10s} {'mean us':>10s} {'share':>7s}"]
for name, t in sorted(tot.items(), key=lambda x: -x[1]):
    lines.append(f"{name[:60]:60s} {cnt[name]:8d} {t / 1000:10.3f} {t / cnt[name]:10.2f} {t / T:7.1%}")
lines.append(f"{'TOTAL':60s} {sum(cnt.values()):8d} {T / 1000:10.3f}")
out = "\n".join(lines)
print(out)
if len(sys.argv) > 2:
    open(sys.argv[2], "w").write(out + "\n")
