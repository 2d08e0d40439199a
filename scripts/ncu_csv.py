"""Print kernel name + duration (us) rows of an ncu --csv launch list (gpu__time_duration.sum)."""
import csv, sys
rows = [l for l in open(sys.argv[1]) if not l.startswith("==")]
r = list(csv.reader(rows))
h = r[0]
ki, vi = h.index("Kernel Name"), h.index("Metric Value")
for row in r[1:]:
    if len(row) > vi:
        print(f"{float(row[vi].replace(',', '')) / 1000:9.1f}  {row[ki][:100]}")
