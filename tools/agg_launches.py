"""Aggregate an ncu --metrics gpu__time_duration.sum CSV launch list by kernel name."""
import csv, collections, re, sys
rows = list(csv.reader(open(sys.argv[1])))
hi = next(i for i, r in enumerate(rows) if 'Kernel Name' in r)
hdr = rows[hi]; ki = hdr.index('Kernel Name'); vi = hdr.index('Metric Value'); ui = hdr.index('Metric Unit')
scale = {'nsecond': 1e-3, 'usecond': 1.0, 'msecond': 1e3, 'ns': 1e-3, 'us': 1.0, 'ms': 1e3}
agg = collections.defaultdict(lambda: [0, 0.0]); tot = 0.0
for r in rows[hi + 1:]:
    if len(r) <= vi: continue
    v = float(r[vi].replace(',', '')) * scale.get(r[ui], 1.0)
    k = re.sub(r'\(.*', '', r[ki])
    k = re.sub(r'^void ', '', k)[:70]
    agg[k][0] += 1; agg[k][1] += v; tot += v
print(f"total {tot/1e3:.2f} ms over {sum(a[0] for a in agg.values())} launches (ncu-serialised, cold)")
for k, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1])[:int(sys.argv[2]) if len(sys.argv) > 2 else 30]:
    print(f"{t/1e3:9.2f} ms {100*t/tot:5.1f}% {c:6d}  {k}")
