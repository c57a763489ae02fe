"""Summarise an ncu --metrics gpu__time_duration.sum CSV launch list."""
import csv, collections, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr = next(i for i, r in enumerate(rows) if 'Kernel Name' in r)
h = rows[hdr]
ki, vi, ui = h.index('Kernel Name'), h.index('Metric Value'), h.index('Metric Unit')
tot, cnt = collections.defaultdict(float), collections.Counter()
scale = {'ns': 1e-6, 'nsecond': 1e-6, 'us': 1e-3, 'usecond': 1e-3, 'ms': 1.0, 'msecond': 1.0, 's': 1e3, 'second': 1e3}
for r in rows[hdr + 1:]:
    if len(r) <= vi:
        continue
    name = r[ki].split('(')[0].replace('void ', '').replace('msot_dev::', '')[:48]
    tot[name] += float(r[vi].replace(',', '')) * scale.get(r[ui], 1e-6)
    cnt[name] += 1
T = sum(tot.values())
print(f"{'ms':>10} {'share':>6} {'count':>6}  kernel")
for k, v in sorted(tot.items(), key=lambda kv: -kv[1])[:int(sys.argv[2]) if len(sys.argv) > 2 else 30]:
    print(f"{v:10.3f} {100 * v / T:5.1f}% {cnt[k]:6d}  {k}")
print(f"{T:10.3f}  total device time of {sum(cnt.values())} launches")
