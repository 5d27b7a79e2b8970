"""Per-CUDA-source-line warp stall samples from an .ncu-rep (source page, cuda,sass)."""
import csv, io, subprocess, sys
from collections import defaultdict

rep, want = sys.argv[1], (sys.argv[2] if len(sys.argv) > 2 else None)
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
per = defaultdict(int)
src = {}
fname = None
hdr = None
cur_line = None
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Function Name":
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None:
        continue
    if r[0]:  # cuda source line row
        cur_line = (fname, int(r[0]))
        src[cur_line] = r[1]
    if len(r) > 4 and r[2]:
        try:
            per[cur_line] += int(r[4] or 0)
        except ValueError:
            pass
tot = sum(per.values()) or 1
for k, v in sorted(per.items(), key=lambda kv: -kv[1])[:int(sys.argv[3]) if len(sys.argv) > 3 else 40]:
    if want and want not in k[0]:
        continue
    print(f"{100*v/tot:5.1f}%  {k[0]}:{k[1]:4d}  {src.get(k, '').strip()[:100]}")
