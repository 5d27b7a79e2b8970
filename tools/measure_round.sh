# Full measurement pass (GPU box): bench (ours + reference arm), bench launch list,
# ncu --set full of the MSDT root GEMMs inside the ALS sweep graphs, the CUPTI
# sweep timeline, and the C5s slice.
cd /root/repo
set -x
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
python bench.py --impl reference > gpurun_out/bench_reference.json 2> gpurun_out/bench_reference.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_bench.csv \
    python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_bench.log 2>&1
python tools/launch_summary.py gpurun_out/launches_bench.csv > gpurun_out/launches_summary.txt
SWEEPS=3 ncu --set full --import-source on --clock-control none -k regex:root_gemm_kernel -c 4 \
    -o gpurun_out/roots_full python tools/profile_als.py > gpurun_out/ncu_roots.log 2>&1
python tools/make_ncu_summary.py gpurun_out/roots_full.ncu-rep gpurun_out/ncu_summary.json \
    "ncu --set full --clock-control none, tools/profile_als.py (C2 ALS sweeps: the three MSDT roots), round 1"
python tools/ncu_summary.py gpurun_out/roots_full.ncu-rep > gpurun_out/ncu_roots_summary.txt
python tools/timeline_als.py > gpurun_out/timeline_als.txt 2>&1
python tools/c5s_smoke.py > gpurun_out/c5s.txt 2>&1
tail -c 400 gpurun_out/bench.json
python tools/timeline_als.py gn > gpurun_out/timeline_gn.txt 2>&1
python tools/gn_breakdown_c5s.py > gpurun_out/c5s_gn.txt 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
tail -1 gpurun_out/smoke.log
