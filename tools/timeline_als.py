"""Real (overlapped) kernel timeline of warm ALS sweeps via CUPTI (torch.profiler):
per-kernel start offsets and durations inside one sweep, and the idle gaps."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from torch.profiler import profile, ProfilerActivity
from paper_1910_12331_b200 import cpkit

mode = sys.argv[1] if len(sys.argv) > 1 else "als"
dims, R, noise = [400, 400, 400], 100, 1e-6
if len(sys.argv) > 2 and sys.argv[2] == "c5s":
    dims, R, noise = [200, 200, 200, 200], 200, 1e-4
truth = cpkit.random_factors(dims, R, cpkit.problem_seed(0, R, 0))
init = cpkit.random_factors(dims, R, cpkit.init_seed(0, R, 0, 0))
p = cpkit.DeviceProblem(dims, R)
p.generate(truth, 1, noise)
p.set_factors(init)
torch.cuda.init()
for _ in range(6):
    p.als_sweep(0.0)
torch.cuda.synchronize()
if mode == "gn":
    p.time_gn_steps({}, 2)  # warm
    p.set_factors(init)
    p.time_gn_steps({}, 1)
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    if mode == "gn":
        p.time_gn_steps({}, 2)
    else:
        p.time_als_sweeps(float(os.environ.get("LAM", "0")), 4 if R < 200 else 2)  # the bench's pipelined loop
    torch.cuda.synchronize()
out = os.path.join(os.environ.get("OUT", "gpurun_out"), f"timeline_{mode}{'_c5s' if R == 200 else ''}.json")
prof.export_chrome_trace(out)
ev = [e for e in json.load(open(out))["traceEvents"] if e.get("cat") == "kernel"]
ev.sort(key=lambda e: e["ts"])
t0 = ev[0]["ts"]
busy_end = t0
for e in ev:
    gap = e["ts"] - busy_end
    name = e["name"].replace("void ", "").replace("cpkit::", "").replace("(anonymous namespace)::", "")
    name = name.split("(")[0][:60]
    print(f"{e['ts'] - t0:9.1f} {e['dur']:7.1f}  gap {gap:6.1f}  s{e['args'].get('stream')}  {name}")
    busy_end = max(busy_end, e["ts"] + e["dur"])
print(f"total span {busy_end - t0:.1f} us ({mode})")
idle = sum(max(0.0, b["ts"] - max(e["ts"] + e["dur"] for e in ev[:i + 1])) for i, b in enumerate(ev[1:]))
print(f"idle (no kernel running) {idle:.1f} us")
