"""Per-kernel totals and shares from an `ncu --metrics gpu__time_duration.sum --csv` launch list."""
import collections
import csv
import signal
import sys

signal.signal(signal.SIGPIPE, signal.SIG_DFL)   # `| head` closes the pipe early: exit quietly

rows = list(csv.reader(open(sys.argv[1])))
hdr = next(i for i, r in enumerate(rows) if 'Kernel Name' in r)
h = rows[hdr]
ki, vi, ui = h.index('Kernel Name'), h.index('Metric Value'), h.index('Metric Unit')
scale = {'ns': 1e-3, 'nsecond': 1e-3, 'us': 1.0, 'usecond': 1.0, 'ms': 1e3, 'msecond': 1e3}
tot, cnt = collections.defaultdict(float), collections.Counter()
for r in rows[hdr + 1:]:
    if len(r) <= vi:
        continue
    name = r[ki].split('(')[0].replace('void ', '').split('<')[0]
    v = float(r[vi].replace(',', '')) * scale.get(r[ui], 1.0)
    tot[name] += v
    cnt[name] += 1
T = sum(tot.values())
print(f"{'kernel':24s} {'launches':>8s} {'total us':>12s} {'us/launch':>10s} {'share':>6s}")
for k, v in sorted(tot.items(), key=lambda x: -x[1]):
    print(f"{k:24s} {cnt[k]:8d} {v:12.1f} {v / cnt[k]:10.1f} {100 * v / T:5.1f}%")
