"""Development: summarise an ncu --csv launch list (gpu__time_duration.sum)."""
import collections
import csv
import io
import re
import sys

lines = [l for l in open(sys.argv[1]) if not l.startswith("==")]
rows = list(csv.DictReader(io.StringIO("".join(lines))))
seq = []
for r in rows:
    v = float(r["Metric Value"].replace(",", ""))
    u = r["Metric Unit"]
    us = v / 1000 if u in ("ns", "nsecond") else (v if u in ("us", "usecond") else v * 1000)
    seq.append((re.sub(r"\(.*", "", r["Kernel Name"])[:56], us, r.get("Grid Size", ""), r.get("Block Size", "")))
if "-s" in sys.argv:
    for s in seq:
        print("%-56s %8.2f %s %s" % s)
agg = collections.defaultdict(lambda: [0, 0.0])
for n, us, _, _ in seq:
    agg[n][0] += 1
    agg[n][1] += us
tot = sum(v[1] for v in agg.values())
print("| kernel | launches | sum us | share |\n|---|---|---|---|")
for n, (c, us) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print("| `%s` | %d | %.1f | %.1f%% |" % (n, c, us, 100 * us / tot))
print("total %.1f us over %d launches" % (tot, len(seq)))
