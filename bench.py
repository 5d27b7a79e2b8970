"""Benchmark of the B200 GN-CG / ALS hot path (BASELINE.json metric).

Workload (BASELINE.json configs[1], "C2"): order-3 tensor, s=400 per mode,
R=100, factors i.i.d. uniform[0,1) from the reference keyed RNG
(problem_seed(0,100,0)), X = reconstruct(truth) + Gaussian noise scaled to
1e-6 ||X||_F, generated on device (512 MB > the 126 MB L2, so no L2 flush is
needed between steps). ALS from a uniform[0,1) init (init_seed(0,100,0,0)).

A step = one ALS sweep (2 root MTTKRP contractions + N SPD solves + grams).
`value` = sweeps/s with the tensor resident in HBM; `e2e` = the same metric
through the public C ABI (host tensor -> device -> optimize -> host factors).
Under torchrun (N>1) the tensor is sharded along its last mode across ranks
(strong scaling of the same C2 problem; NCCL all-reduce / all-gather of the
s x R MTTKRP partials over NVLink).

--impl reference times the reference algorithm's CPU path (the oracle
restatement, oracle/, all host threads) on the same workload.
"""
import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

DIMS = [400, 400, 400]
RANK = 100
NOISE = 1e-6
METRIC = "ALS sweeps/s (order-3 s=400 R=100, C2)"
UNIT = "sweeps/s"
E2E_SWEEPS = 20


def workload_config(world):
    return {"workload": "C2: order-3 s=400 R=100 uniform[0,1) exact rank + 1e-6 noise, ALS",
            "dims": DIMS, "rank": RANK, "noise_rel": NOISE, "master_seed": 0,
            "step": "one ALS sweep", "l2": "tensor 512 MB > 126 MB L2 (no flush needed)",
            "parallelism": f"last-mode shard x{world}" if world > 1 else "single GPU",
            "sharding": "mode-3 slabs, NCCL allreduce/allgather of s x R partials"}


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = "clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown," \
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown," \
             "clocks_event_reasons.sw_power_cap"

    def __init__(self, device):
        self.device = device
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "20"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None
        time.sleep(0.15)
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx = max(mx, float(parts[1]))
            except ValueError:
                continue
            for n, v in zip(names, parts[3:7]):
                if v.lower() in ("active", "1"):
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx or None,
                "samples": len(sm), "reasons": sorted(reasons)}


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f)
    except OSError:
        return {}


def ncu_traffic():
    """Per-launch DRAM bytes of the root GEMMs from the committed ncu --set full capture."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_summary.json")) as f:
            return json.load(f)
    except OSError:
        return {}


# ------------------------------------------------------------------------ reference arm
def run_reference(args, rank, world):
    if rank != 0:
        return 0
    from oracle import oracle as orc
    cores = os.cpu_count() or 1
    orc.set_threads(cores)
    t0 = time.time()
    truth = orc.random_model(DIMS, RANK, orc.problem_seed(0, RANK, 0))
    x = orc.reconstruct(truth)
    xn = float(np.linalg.norm(x))
    noise = np.random.default_rng(0x4E01).standard_normal(x.shape)  # timing input only
    x += NOISE * xn / float(np.linalg.norm(noise)) * noise
    del noise
    init = orc.random_model(DIMS, RANK, orc.init_seed(0, RANK, 0, 0))
    gen_s = time.time() - t0
    f = init
    for _ in range(args.warmup):
        f, _, _, _ = orc.als_sweep(x, f, 0.0)
    times = []
    for _ in range(args.steps):
        t = time.perf_counter()
        f, _, _, _ = orc.als_sweep(x, f, 0.0)
        times.append(time.perf_counter() - t)
    total = sum(times)
    value = args.steps / total
    out = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * total / args.steps,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded keyed-RNG factors; numpy Gaussian noise for the CPU timing input)",
        "config": workload_config(1),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "port",
                         "sample": f"{args.steps} ALS sweeps of the full C2 tensor (oracle restatement "
                                   f"of als.cpp:22-52, {cores} threads); input generation {gen_s:.1f}s untimed"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "note": "reference (Eigen/CMake) cannot be built here; oracle/ is its CPU restatement",
    }
    print(json.dumps(out), flush=True)
    return 0


# ------------------------------------------------------------------------ B200 arm
def cpu_baseline_sample(x_host, init):
    """Oracle ALS sweep on the host cores over the same tensor (reported only).
    Two settings: all host cores (the reported value), and one
    thread, the reference's own setting (Eigen without OpenMP)."""
    from oracle import oracle as orc
    cores = os.cpu_count() or 1
    orc.set_threads(cores)
    t = time.perf_counter()
    orc.als_sweep(x_host, init, 0.0)
    dt = time.perf_counter() - t
    orc.set_threads(1)
    t = time.perf_counter()
    orc.als_sweep(x_host, init, 0.0)
    dt1 = time.perf_counter() - t
    orc.set_threads(cores)
    return {"value": 1.0 / dt, "unit": UNIT, "cores": cores, "kind": "port",
            "sample": f"1 ALS sweep of the full C2 tensor (oracle restatement of als.cpp:22-52, "
                      f"{cores} threads, {dt:.2f}s)",
            "single_thread": {"value": 1.0 / dt1, "unit": UNIT, "cores": 1,
                              "sample": f"the same sweep on 1 thread, the reference's setting ({dt1:.2f}s)"}}


def run_b200(args, rank, world, local_rank):
    from paper_1910_12331_b200 import cpkit
    cpkit.load()
    dist = None
    nccl_id = None
    if world > 1:
        import torch
        import torch.distributed as tdist
        torch.cuda.set_device(local_rank)
        tdist.init_process_group("nccl")
        dist = tdist
        buf = torch.zeros(128, dtype=torch.uint8, device="cuda")
        if rank == 0:
            buf.copy_(torch.frombuffer(bytearray(cpkit.nccl_unique_id()), dtype=torch.uint8))
        tdist.broadcast(buf, 0)
        nccl_id = bytes(buf.cpu().numpy().tobytes())

    def barrier():
        if dist:
            dist.barrier()

    def max_over_ranks(v):
        if not dist:
            return v
        import torch
        t = torch.tensor([v], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    truth = cpkit.random_factors(DIMS, RANK, cpkit.problem_seed(0, RANK, 0))
    init = cpkit.random_factors(DIMS, RANK, cpkit.init_seed(0, RANK, 0, 0))
    p = cpkit.DeviceProblem(DIMS, RANK, device=local_rank, shard=rank, world=world, nccl_id=nccl_id)
    p.generate(truth, noise_seed=1, noise_rel=NOISE)
    p.set_factors(init)
    lo, hi, local_elems = p.slab()

    peak_dmma = cpkit.probe_dmma_peak(local_rank)

    # ---- warm-up, then exactly K timed sweeps (CUDA events on the problem's stream);
    # clocks are sampled from just before the warm-up through the timed region
    with ClockSampler(local_rank) as clk:
        p.time_als_sweeps(0.0, max(1, args.warmup))
        p.set_factors(init)
        barrier()
        launches0 = cpkit.kernel_launches()
        p.profile(True)
        ms = p.time_als_sweeps(0.0, args.steps)
        prof_ms, prof_cnt = p.profile_read()
        p.profile(False)
        launches = cpkit.kernel_launches() - launches0
    barrier()
    ms = max_over_ranks(ms)
    value = args.steps / (ms / 1e3)

    # ---- roofline: root MTTKRP GEMMs (2 per sweep), measured inside the timed region
    flops_per_root = 2.0 * RANK * local_elems
    root_ms = (prof_ms[0] + prof_ms[1]) / max(1, prof_cnt[0] + prof_cnt[1])
    achieved_tf = flops_per_root / (root_ms * 1e-3) / 1e12
    share = (prof_ms[0] + prof_ms[1]) / ms if ms > 0 else None
    traffic = ncu_traffic().get("root_gemm_dram_bytes_per_launch")  # committed ncu --set full capture

    # ---- secondary kernels: J^T J v (GN inner loop) and ||X||^2 streaming
    peaks = measured_peaks()
    hbm = peaks.get("hbm_gbs", 6650.0)
    jtj_ms = p.time_jtj(50)
    S = sum(DIMS)
    jtj_bytes = 8.0 * (3 * RANK * S + len(DIMS) * (len(DIMS) + 1) / 2 * RANK * RANK)
    jtj_flops = 6.0 * RANK * RANK * S
    nrm_ms = p.time_norm2(5)
    nrm_gbs = 8.0 * local_elems / (nrm_ms * 1e-3) / 1e9
    # the same streaming kernel on a >= 1 GB tensor (bandwidth-bound
    # kernels shown at a size where HBM, not launch latency, is the bound)
    big = None
    if world == 1:
        bdims = [512, 512, 512]  # 1.07 GB
        pb = cpkit.DeviceProblem(bdims, 1)
        pb.generate(cpkit.random_factors(bdims, 1, 7))
        big_ms = pb.time_norm2(10)
        big_bytes = 8.0 * 512 ** 3
        big = {"ms": big_ms, "gbs": big_bytes / (big_ms * 1e-3) / 1e9, "bytes": big_bytes}
        pb.close()

    # ---- GN outer iterations (default config: varying lambda, CG cap min(sum s R, 10 R)=1000)
    # GN: steady-state iterations. Each timed call starts from the same init with
    # the tree pass of the starting point already cached (gn_optimize computes it
    # once before its first iteration), so the per-iteration figure is one tree
    # pass (the post-step residual) + gradient + preconditioner + CG + update.
    GN_STEPS = 4
    gn_runs = []
    for i in range(4):  # first call warms the CG kernel's launch path; median of the rest
        p.set_factors(init)  # time_gn_steps caches the starting point's tree pass before timing
        gn_runs.append(p.time_gn_steps({}, GN_STEPS))
    gn_ms = statistics.median(r[0] for r in gn_runs[1:])
    gn_cg = gn_runs[-1][1]

    # ---- end to end through the public C ABI (host tensor in, host factors out)
    import torch
    x_pinned = torch.empty(local_elems, dtype=torch.float64, pin_memory=True).numpy()
    p.download_into(x_pinned)
    e2e_cfg = {"optimizer": "als", "als": {"max_sweeps": E2E_SWEEPS, "residual_tol": 0.0,
                                           "step_tol": 0.0}}
    e2e_times = []
    for i in range(max(1, args.e2e_steps) + 1):
        barrier()
        t = time.perf_counter()
        p.upload(x_pinned)
        out, rep = p.optimize(e2e_cfg, init)
        dt = time.perf_counter() - t
        if i > 0:
            e2e_times.append(dt)
    e2e_dt = max_over_ranks(statistics.median(e2e_times))
    e2e_value = E2E_SWEEPS / e2e_dt
    final = rep.to_json()["records"][-1]

    result = None
    if rank == 0:
        result = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (reference keyed RNG, generated on device)",
            "config": workload_config(world),
            "roofline": {"bound": "tensor", "kernel": "root MTTKRP GEMM (TMA + DMMA m16n8k16)",
                         "achieved": achieved_tf, "peak": peak_dmma, "unit": "TFLOP/s",
                         "frac": achieved_tf / peak_dmma,
                         "peak_source": "FP64 DMMA issue-rate probe measured in this run "
                                        "(MEASURED_PEAKS.json has no fp64 entry)",
                         "traffic": traffic, "algorithmic_flops_per_launch": flops_per_root,
                         "algorithmic_bytes_per_launch": 8.0 * local_elems + 8.0 * RANK * 160000,
                         "avg_launch_ms": root_ms, "launches": prof_cnt[0] + prof_cnt[1],
                         "share_of_step": share},
            "kernels": {
                "jtj_matvec": {"ms": jtj_ms, "gbs": jtj_bytes / (jtj_ms * 1e-3) / 1e9,
                               "hbm_frac": jtj_bytes / (jtj_ms * 1e-3) / 1e9 / hbm,
                               "tflops": jtj_flops / (jtj_ms * 1e-3) / 1e12,
                               "bytes": jtj_bytes, "note": "3.4 MB working set, L2-resident, launch-bound"},
                "norm2_1GB": None if big is None else {**big, "hbm_frac": big["gbs"] / hbm},
                "norm2": {"ms": nrm_ms, "gbs": nrm_gbs, "hbm_frac": nrm_gbs / hbm,
                          "peak_gbs": hbm, "peak_source": "MEASURED_PEAKS.json hbm_gbs"},
            },
            "gn": {"iters_per_s": GN_STEPS / (gn_ms * 1e-3), "ms_per_iter": gn_ms / GN_STEPS,
                   "cg_iters_total": gn_cg, "iters": GN_STEPS,
                   "config": "default GnConfig (varying lambda, cg cap 1000), steady state: "
                             "the starting point's tree pass cached before timing"},
            "e2e": {"value": e2e_value, "unit": UNIT,
                    "h2d_bytes_per_step": int(8 * local_elems + 8 * S * RANK),
                    "d2h_bytes_per_step": int(8 * S * RANK),
                    "path": f"cpkit_dev_upload_tensor + cpkit_dev_optimize (ALS, {E2E_SWEEPS} sweeps) "
                            "+ host factors", "final_fitness": final["fitness"]},
            "gpu_launches": int(launches),
            "clocks": clk.summary(),
        }
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        x_host = x_pinned.reshape(DIMS)
        result["cpu_baseline"] = cpu_baseline_sample(x_host, init)
    p.close()
    if rank == 0 and world == 1 and not args.no_c5s:
        result["c5s"] = c5s_slice(cpkit, result["roofline"]["peak"])
    if dist:
        dist.destroy_process_group()
    if rank == 0:
        print(json.dumps(result), flush=True)
    return 0


def c5s_slice(cpkit, peak_tf):
    """The largest config that fits one GPU (C5s: order 4, s=200, R=200, 12.8 GB,
    the 1-GPU anchor of the C5 scaling case), generated on device: ALS sweep and
    GN iteration times, reported beside the headline (not the bench value)."""
    dims, R = [200] * 4, 200
    truth = cpkit.random_factors(dims, R, cpkit.problem_seed(0, R, 0))
    init = cpkit.random_factors(dims, R, cpkit.init_seed(0, R, 0, 0))
    q = cpkit.DeviceProblem(dims, R)
    q.generate(truth, 1, 1e-4)
    q.set_factors(init)
    q.time_als_sweeps(0.0, 1)  # warm-up (graph capture)
    als_ms = q.time_als_sweeps(0.0, 3) / 3
    q.set_factors(init)
    q.time_gn_steps({}, 1)  # warm-up
    q.set_factors(init)
    gn_ms, cg = q.time_gn_steps({}, 2)
    q.close()
    root_flops = 4.0 * R * 200 ** 4  # two root contractions per sweep / per GN iteration
    return {"workload": "C5s: order-4 s=200 R=200 uniform[0,1) + 1e-4 noise (12.8 GB), generated on device",
            "als_ms_per_sweep": als_ms, "als_sweeps_per_s": 1e3 / als_ms,
            "als_root_tflops": root_flops / (als_ms * 1e-3) / 1e12,
            "als_root_frac_of_peak": root_flops / (als_ms * 1e-3) / 1e12 / peak_tf,
            "gn_ms_per_iter": gn_ms / 2, "gn_cg_iters": cg,
            "note": "TFLOP/s = the two root contractions' 4 R prod(s) flops over the whole sweep time"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-c5s", action="store_true", help="skip the C5s (largest single-GPU config) line item")
    args = ap.parse_args()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        return run_reference(args, rank, world)
    return run_b200(args, rank, world, local_rank)


if __name__ == "__main__":
    sys.exit(main())
