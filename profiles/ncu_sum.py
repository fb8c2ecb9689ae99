"""Mean kernel duration (us) and launch count per kernel from an ncu --csv launch list."""
import collections
import csv
import sys

for f in sys.argv[1:]:
    rows = [r for r in csv.reader(open(f)) if len(r) > 10]
    h = next(r for r in rows if "Kernel Name" in r)
    k, m = h.index("Kernel Name"), h.index("Metric Value")
    d = collections.defaultdict(list)
    for r in rows[rows.index(h) + 1:]:
        d[r[k].split("(")[0][:40]].append(float(r[m].replace(",", "")))
    print(f, {n: (round(sum(x) / len(x) / 1e3, 2), len(x)) for n, x in d.items()})
