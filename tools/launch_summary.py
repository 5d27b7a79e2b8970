"""Aggregate an ncu --csv launch list (gpu__time_duration.sum): per-kernel totals; optional last-N launches."""
import csv, collections, sys
rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
h = rows[0]
ik, iv, iu = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
seq = []
for r in rows[1:]:
    v = float(r[iv].replace(",", ""))
    us = {"nsecond": v / 1e3, "usecond": v, "msecond": v * 1e3}.get(r[iu], v / 1e3)
    seq.append((r[ik].split("(")[0].replace("void ", "").replace("cpkit::", "").replace("<unnamed>::", "")[-70:], us))
last = int(sys.argv[2]) if len(sys.argv) > 2 else len(seq)
seq = seq[-last:]
agg = collections.defaultdict(lambda: [0, 0.0])
for n, us in seq:
    agg[n][0] += 1
    agg[n][1] += us
tot = sum(a[1] for a in agg.values())
print(f"{len(seq)} launches, {tot:.1f} us total")
for k, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{t:9.1f} us {c:4d}x  {k}")
