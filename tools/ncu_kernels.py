"""Per-kernel summary of an `ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,
dram__bytes_write.sum,dram__throughput.avg.pct_of_peak_sustained_elapsed,
sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active --csv --log-file X` run:
launches, mean duration, DRAM bytes per launch, achieved GB/s, % of DRAM peak,
tensor-pipe %.   python tools/ncu_kernels.py X.csv [header line]"""
import collections
import csv
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
h = rows[0]
ki, mi, vi, ui, idi = (h.index(k) for k in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit", "ID"))
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9, "ns": 1e-9, "usecond": 1e-6,
         "us": 1e-6, "msecond": 1e-3, "ms": 1e-3}
per = collections.defaultdict(dict)
names = {}
for r in rows[1:]:
    per[r[idi]][r[mi]] = float(r[vi].replace(",", "")) * scale.get(r[ui], 1)
    names[r[idi]] = r[ki].split("(")[0].replace("(anonymous namespace)::", "")[:52]
agg = collections.defaultdict(lambda: [0, 0.0, 0.0, 0.0, 0.0])
for i, d in per.items():
    a = agg[names[i]]
    a[0] += 1
    a[1] += d.get("gpu__time_duration.sum", 0)
    a[2] += d.get("dram__bytes_read.sum", 0) + d.get("dram__bytes_write.sum", 0)
    a[3] += d.get("dram__throughput.avg.pct_of_peak_sustained_elapsed", 0)
    a[4] += d.get("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", 0)
if len(sys.argv) > 2:
    print(sys.argv[2])
for k, (n, t, b, pct, tp) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"{k:52s} n={n:3d} avg {t / n * 1e6:8.1f} us  DRAM {b / n / 1e6:8.1f} MB/launch "
          f"{b / t / 1e9 if t else 0:7.1f} GB/s  dram% {pct / n:5.1f}  tensor% {tp / n:5.1f}")
