"""Summarise an .ncu-rep: per kernel duration, DRAM bytes, DMMA pipe %, top stall sources."""
import csv, io, subprocess, sys

rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr = rows[0]
keys = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
        "sm__warps_active.avg.pct_of_peak_sustained_active",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum"]
units = rows[1]
for r in rows[2:]:
    d = dict(zip(hdr, r))
    print("==", d["Kernel Name"][:90])
    print("   " + "  ".join(f"{k.split('.')[0].split('__')[-1]}={d.get(k,'?')}{units[hdr.index(k)] if k in hdr else ''}" for k in keys))
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
kern = []
cur = None
for r in csv.reader(io.StringIO(src)):
    if r and r[0] == "Kernel Name":
        cur = {"name": r[1], "rows": []}
        kern.append(cur)
    elif r and r[0] == "Address":
        cur["hdr"] = r
    elif cur is not None and r:
        cur["rows"].append(r)
seen = set()
for k in kern:
    if k["name"] in seen:
        continue
    seen.add(k["name"])
    h = k["hdr"]
    i_s, i_src = h.index("Warp Stall Sampling (All Samples)"), h.index("Source")
    tot = sum(int(r[i_s]) for r in k["rows"]) or 1
    print("-- top stall lines:", k["name"][:70])
    for r in sorted(k["rows"], key=lambda r: -int(r[i_s]))[:int(sys.argv[2]) if len(sys.argv) > 2 else 8]:
        print(f"   {100*int(r[i_s])/tot:5.1f}%  {r[i_src].strip()[:80]}")
