"""Per-source-line stall samples split by stall reason (source page cuda,sass)."""
import csv, io, subprocess, sys
from collections import defaultdict

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
kfilt = sys.argv[3] if len(sys.argv) > 3 else None
active = kfilt is None
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
per = defaultdict(lambda: defaultdict(int))
src, fname, hdr, cur = {}, None, None, None
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]; continue
    if r[0] == "Function Name":
        active = kfilt is None or kfilt in r[1]
        continue
    if not active:
        continue
    if r[0] == "Line No":
        hdr = r; continue
    if hdr is None:
        continue
    if r[0]:
        cur = (fname, int(r[0])); src[cur] = r[1]
    if len(r) > 4 and r[2] and r[2] != "...":
        for i, h in enumerate(hdr):
            if h.startswith("stall_") and i < len(r):
                try:
                    per[cur][h[6:]] += int(float(r[i] or 0))
                except ValueError:
                    pass
tot = sum(sum(v.values()) for v in per.values()) or 1
for k, v in sorted(per.items(), key=lambda kv: -sum(kv[1].values()))[:top]:
    s = sum(v.values())
    reasons = ", ".join(f"{a}={100*b/s:.0f}%" for a, b in sorted(v.items(), key=lambda x: -x[1])[:3] if b)
    print(f"{100*s/tot:5.1f}%  {k[0]}:{k[1]:4d}  [{reasons}]  {src.get(k, '').strip()[:70]}")
