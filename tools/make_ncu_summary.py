"""Write profiles/ncu_summary.json from an ncu --set full capture of the root GEMMs
(tools/profile_roots.py). bench.py reads root_gemm_dram_bytes_per_launch from it
for roofline.traffic."""
import csv, io, json, subprocess, sys

rep, out, label = sys.argv[1], sys.argv[2], sys.argv[3] if len(sys.argv) > 3 else ""
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units = rows[0], rows[1]


def val(d, k):
    v = d.get(k, "")
    try:
        x = float(v.replace(",", ""))
    except ValueError:
        return None
    u = units[hdr.index(k)] if k in hdr else ""
    scale = {"Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "byte": 1.0, "usecond": 1e-6, "msecond": 1e-3,
             "nsecond": 1e-9, "second": 1.0, "us": 1e-6, "ms": 1e-3, "ns": 1e-9, "s": 1.0,
             "KB": 1e3, "MB": 1e6, "GB": 1e9, "B": 1.0}.get(u, 1.0)
    return x * scale


kernels = []
for r in rows[2:]:
    d = dict(zip(hdr, r))
    if "root_gemm_" not in d.get("Kernel Name", ""):
        continue
    kernels.append({
        "kernel": d["Kernel Name"][:90],
        "duration_s": val(d, "gpu__time_duration.sum"),
        "dram_read_bytes": val(d, "dram__bytes_read.sum"),
        "dram_write_bytes": val(d, "dram__bytes_write.sum"),
        "dmma_pipe_active_pct": val(d, "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active"),
        "registers": d.get("launch__registers_per_thread"),
        "grid": d.get("launch__grid_size"),
        "block": d.get("launch__block_size"),
    })
# One root contraction = a main launch plus, when the tiles leave a partial last
# wave, its split-K tail launch (plan_back). Traffic per contraction = all
# captured root-kernel DRAM bytes / number of main launches (the long ones).
longest = max(k["duration_s"] for k in kernels)
mains = [k for k in kernels if k["duration_s"] >= 0.5 * longest]
total = sum(k["dram_read_bytes"] + k["dram_write_bytes"] for k in kernels)
summary = {"source": label or "ncu --set full --clock-control none (root GEMMs)",
           "kernels": kernels,
           "root_gemm_dram_bytes_per_launch": total / len(mains),
           "note": "per root contraction (main launch + its split-K tail launch when present)"}
with open(out, "w") as f:
    json.dump(summary, f, indent=1)
print(json.dumps(summary, indent=1))
