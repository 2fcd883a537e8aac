"""Hot SASS regions of one ncu report (--page source): python scripts/ncu_hot.py REP [NBLK] [SPAN]
prints the top blocks of SPAN consecutive instructions by executed warp instructions and stall samples."""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
nblk = int(sys.argv[2]) if len(sys.argv) > 2 else 12
span = int(sys.argv[3]) if len(sys.argv) > 3 else 24
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[1]
data = rows[2:]
isrc, ie, iss, ith = (h.index(x) for x in ("Source", "Instructions Executed", "Warp Stall Sampling (All Samples)",
                                          "Avg. Threads Executed"))
tot = sum(int(r[ie]) for r in data)
st = sum(int(r[iss]) for r in data)
print(f"total warp instructions {tot}, stall samples {st}")
agg = []
for k in range(0, len(data), span):
    blk = data[k:k + span]
    agg.append((sum(int(r[ie]) for r in blk), sum(int(r[iss]) for r in blk), k))
agg.sort(reverse=True)
for a in agg[:nblk]:
    print(f"{a[0]:>12d} {100.0 * a[0] / tot:5.1f}% samples {100.0 * a[1] / st:5.1f}%  @{a[2]:5d} {data[a[2]][isrc].strip()[:50]}")
if len(sys.argv) > 4:
    lo, hi = (int(x) for x in sys.argv[4].split(":"))
    for k in range(lo, hi):
        r = data[k]
        print(k, r[ie].rjust(10), r[iss].rjust(6), r[ith].rjust(5), r[isrc].strip()[:80])
