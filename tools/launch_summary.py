"""Summarise an ncu --metrics gpu__time_duration.sum launch list (CSV):
per kernel: launches, mean and total duration, share."""
import csv, sys, collections
rows = list(csv.reader(open(sys.argv[1])))
h = next(i for i, r in enumerate(rows) if 'Kernel Name' in r)
hdr = rows[h]; ki = hdr.index('Kernel Name'); vi = hdr.index('Metric Value')
d = collections.defaultdict(list)
for r in rows[h + 1:]:
    if len(r) > vi:
        try:
            d[r[ki].split('(')[0][:48]].append(float(r[vi].replace(',', '')))
        except ValueError:
            pass
tot = sum(sum(v) for v in d.values())
for k, v in sorted(d.items(), key=lambda kv: -sum(kv[1])):
    print(f"{k:48s} n={len(v):6d} mean={sum(v)/len(v)/1e3:9.3f} us total={sum(v)/1e6:9.2f} ms share={sum(v)/tot:6.1%}")
