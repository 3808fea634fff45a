"""Print (kernel, gpu__time_duration) rows of an `ncu --csv --log-file` launch list."""
import csv
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
h = rows[0]
ki, vi = h.index("Kernel Name"), h.index("Metric Value")
for r in rows[1:]:
    print(f"{r[vi]:>12}  {r[ki][:100]}")
