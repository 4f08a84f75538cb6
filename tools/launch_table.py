"""Summarise an ncu launch-list CSV (gpu__time_duration.sum): launches and mean us per kernel."""
import collections
import csv
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
h = rows[0]
ik, iv = h.index("Kernel Name"), h.index("Metric Value")
d = collections.OrderedDict()
for r in rows[1:]:
    d.setdefault(r[ik][:70], []).append(float(r[iv].replace(",", "")))
for k, v in d.items():
    print(f"{k:70s} {len(v):4d} {sum(v) / len(v) / 1e3:10.1f} us")
