"""Per-kernel durations (µs) from an ncu --metrics gpu__time_duration.sum --csv launch list."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
h = next(i for i, r in enumerate(rows) if 'Kernel Name' in r)
hdr = rows[h]
ki, vi, ii = hdr.index('Kernel Name'), hdr.index('Metric Value'), hdr.index('ID')
lim = int(sys.argv[2]) if len(sys.argv) > 2 else 10**9
for r in rows[h + 1:]:
    if len(r) <= vi or int(r[ii]) >= lim:
        continue
    print(f"{r[ii]:>4} {float(r[vi].replace(',', '')) / 1e3:10.1f}  {r[ki][:70]}")
