"""Summarise an `ncu --metrics gpu__time_duration.sum --csv --log-file` launch
list: total time per kernel (template arguments kept), share, launch count."""
import collections
import csv
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
h = rows[0]
ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
tot = collections.defaultdict(float)
cnt = collections.Counter()
for r in rows[1:]:
    scale = {"nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0}.get(r[ui], 1e-6)
    name = r[ki].replace("(anonymous namespace)::", "").replace("hzp::", "")
    name = name.split("(")[0] if "gemm_tc_kernel" not in name else name.split(">(")[0] + ">"
    tot[name] += float(r[vi].replace(",", "")) * scale
    cnt[name] += 1
total = sum(tot.values())
print(f"total {total:.2f} ms over {sum(cnt.values())} launches")
for k, v in sorted(tot.items(), key=lambda kv: -kv[1]):
    print(f"{v:9.2f} ms {100 * v / total:5.1f}%  n={cnt[k]:5d}  {k[:110]}")
