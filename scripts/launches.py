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
    name = r[ki].replace('<unnamed>::', 'alu-bench::').split('(')[0].replace('void ', '').split('<')[0]
    v = float(r[vi].replace(',', '')) * scale.get(r[ui], 1.0)
    tot[name] += v
    cnt[name] += 1
# not part of a step: the ALU micro-benchmark (bench.py alu_peak) and the handle's creation
# (exact build, wall normals, host-order scatter)
OFF = ('alu-bench::', 'sb::k_build_cells', 'sb::k_normals', 'sb::k_from_ids')
T = sum(tot.values())
Ts = sum(v for k, v in tot.items() if not k.startswith(OFF))
print(f"{'kernel':24s} {'launches':>8s} {'total us':>12s} {'us/launch':>10s} {'share':>6s} {'of step':>7s}")
for k, v in sorted(tot.items(), key=lambda x: -x[1]):
    st = '      -' if k.startswith(OFF) else f"{100 * v / Ts:6.1f}%"
    print(f"{k:24s} {cnt[k]:8d} {v:12.1f} {v / cnt[k]:10.1f} {100 * v / T:5.1f}% {st}")
print(f"('of step' excludes {', '.join(OFF)}: the ALU micro-benchmark and the handle's creation)")
