"""Aggregate an ncu --metrics gpu__time_duration.sum launch list (CSV)."""
import csv, collections, sys
rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if 'Kernel Name' in r][0]
hdr = rows[hi]; k = hdr.index('Kernel Name'); v = hdr.index('Metric Value')
agg = collections.OrderedDict(); cnt = collections.Counter()
for r in rows[hi + 1:]:
    if len(r) <= v: continue
    name = r[k].split('(')[0].replace('tc::', '').replace('<unnamed>::', '')[-60:]
    t = float(r[v].replace(',', ''))
    agg[name] = agg.get(name, 0) + t; cnt[name] += 1
tot = sum(agg.values())
for n, t in sorted(agg.items(), key=lambda x: -x[1])[:int(sys.argv[2]) if len(sys.argv) > 2 else 25]:
    print("%10.1f us %5.1f%% %4d  %8.1f us/launch  %s" % (t / 1e3, 100 * t / tot, cnt[n], t / 1e3 / cnt[n], n))
