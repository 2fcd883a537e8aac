import csv, collections, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr = next(i for i, r in enumerate(rows) if 'Kernel Name' in r)
h = rows[hdr]; ki = h.index('Kernel Name'); vi = h.index('Metric Value'); ui = h.index('Metric Unit')
tot = collections.defaultdict(float); cnt = collections.Counter()
for r in rows[hdr + 1:]:
    if len(r) <= vi: continue
    name = r[ki].split('(')[0].replace('void ', '').split('<')[0]
    v = float(r[vi].replace(',', '')); u = r[ui]
    v = v / 1e3 if u == 'nsecond' else (v * 1e3 if u == 'msecond' else v)
    tot[name] += v; cnt[name] += 1
T = sum(tot.values())
for k, v in sorted(tot.items(), key=lambda x: -x[1]):
    print(f"{k:28s} {cnt[k]:5d} launches {v:10.1f} us total {v/cnt[k]:9.1f} us/launch {100*v/T:5.1f}%")
